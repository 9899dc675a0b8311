"""Cost-model calibration plumbing on CPU: the samples CSV round-trips through the reference-shaped
reader (cost_model.cpp:105-123 contract: header, comments, separators, malformed-line error), and
the fit of those samples equals the compiled reference's fit_linear bit for bit."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_21257_b200 import calibrate
from paper_2603_21257_b200 import tiersim as t


def test_samples_csv_round_trip_and_reader_contract(tmp_path):
    rng = np.random.default_rng(0)
    samples = [(int(n), float(2.4e-6 * n + 1e-4 + rng.normal(0, 1e-5))) for n in rng.integers(256, 120000, 50)]
    p = tmp_path / "s.csv"
    t.write_samples_csv(p, samples)
    back = t.read_samples_csv(p)
    assert [(s.tokens, s.seconds) for s in back] == samples  # 17 significant digits: exact doubles
    q = tmp_path / "mixed.csv"
    q.write_text("# measured on B200\ntokens;seconds\n\n256\t0.001\n512 ; 0.002\n768,0.003\n")
    assert [(s.tokens, s.seconds) for s in t.read_samples_csv(q)] == [(256, 0.001), (512, 0.002), (768, 0.003)]
    bad = tmp_path / "bad.csv"
    bad.write_text("tokens,seconds\n256,0.001\noops\n")
    with pytest.raises(t.Error, match=r"read_samples_csv: malformed line in .*bad.csv: oops"):
        t.read_samples_csv(bad)
    with pytest.raises(t.Error, match="read_samples_csv: cannot open"):
        t.read_samples_csv(tmp_path / "missing.csv")


def test_fit_of_csv_samples_equals_reference(tmp_path, ref_lib):
    rng = np.random.default_rng(3)
    tok = rng.integers(256, 130000, 200).astype(np.int64)
    sec = 2.38e-6 * tok + 3e-4 + rng.normal(0, 2e-5, 200)
    t.write_samples_csv(tmp_path / "x.csv", zip(tok.tolist(), sec.tolist()))
    s = t.read_samples_csv(tmp_path / "x.csv")
    fit = t.fit_linear((x.tokens, x.seconds) for x in s)
    out = (C.c_double * 4)()
    tk = np.array([x.tokens for x in s], np.int64)
    sc = np.array([x.seconds for x in s], np.float64)
    assert ref_lib.ref_fit_linear(len(s), tk.ctypes.data, sc.ctypes.data, out) == 0
    assert (fit.model.slope, fit.model.intercept) == (out[0], out[1])


def test_calibration_from_stage_requests(tmp_path):
    """The request rows a stage run returns -> CSVs -> fitted models (no device: synthetic rows)."""
    dt = np.dtype([("pick_position", np.int32), ("deferred_chunks", np.int32), ("chunks", np.int64),
                   ("cached_tokens", np.int64), ("compute_tokens", np.int64),
                   ("ingest_begin_ms", np.float64), ("resident_ms", np.float64), ("done_ms", np.float64)])
    n = 40
    rows = np.zeros(n, dt)
    rng = np.random.default_rng(1)
    rows["chunks"] = rng.integers(0, 400, n)
    rows["cached_tokens"] = rows["chunks"] * 256
    rows["compute_tokens"] = rng.integers(30, 4000, n)
    rows["ingest_begin_ms"] = np.arange(n) * 100.0
    rows["resident_ms"] = rows["ingest_begin_ms"] + (2.4e-6 * rows["cached_tokens"] + 5e-4) * 1e3
    rows["pick_position"] = np.arange(n)
    # a request whose reservation waited for a release: its span includes the wait, not a T_load sample
    rows["deferred_chunks"][3] = 5
    rows["resident_ms"][3] += 500.0
    # prefills queue on one compute stream: request k starts at max(resident_k, done_{k-1})
    prev = 0.0
    for k in range(n):
        start = max(rows["resident_ms"][k], prev)
        rows["done_ms"][k] = start + (1e-5 * rows["compute_tokens"][k] + 2e-3) * 1e3
        prev = rows["done_ms"][k]

    class R:
        requests = rows

    cfg = t.ClusterConfig()
    cal = calibrate.calibrate(R(), cfg, str(tmp_path), fit_compute=True)
    assert abs(cal.models.load.slope - 2.4e-6) / 2.4e-6 < 1e-9 and abs(cal.models.load.intercept - 5e-4) < 1e-12
    assert abs(cal.models.comp.slope - 1e-5) / 1e-5 < 1e-9 and abs(cal.models.comp.intercept - 2e-3) < 1e-12
    assert cal.default.load.slope == t.cost_models_from_config(cfg).load.slope
    assert len(t.read_samples_csv(cal.load_csv)) == int(((rows["chunks"] > 0) & (rows["deferred_chunks"] == 0)).sum())
