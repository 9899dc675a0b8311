"""bench.py contract pieces that run without a GPU: the reference arm (--impl reference, the oracle
port on the host cores) prints one JSON line with the contract keys without loading the product
library, exits 0 on a non-zero rank without output, and `--gpus N` launches N ranks itself."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}
ARGS = ["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-chunks-per-request", "1",
        "--workload", "llama8b32k"]


def _run(env_extra, extra=()):
    env = dict(os.environ, **env_extra)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        if k not in env_extra:
            env.pop(k, None)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *ARGS, *extra],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    p = _run({})
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"] == "llama3.1-8b_1x32k" and line["n_gpus"] == 1


def test_reference_arm_other_ranks_exit_silently():
    p = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_gpus_n_self_launches_ranks():
    """`python bench.py --gpus 2` without torchrun: two ranks start (torch.distributed.run on
    127.0.0.1), rank 0 alone prints one line that reports n_gpus = 2."""
    p = _run({}, ["--gpus", "2"])
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_reference_arm_never_loads_the_product():
    """The CPU arm imports numpy + oracle/ only: no paper_2603_21257_b200 module, no libtsb.so."""
    code = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', {', '.join(repr(a) for a in ARGS)}]\n"
        f"runpy.run_path({str(ROOT / 'bench.py')!r}, run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "bad = [m for m in sys.modules if m.startswith('paper_2603_21257_b200')]\n"
        "print(json.dumps({'modules': bad, 'libtsb': 'libtsb.so' in maps}))\n"
    )
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    assert got == {"modules": [], "libtsb": False}


def test_specs_equal_product_workloads():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2603_21257_b200.workloads import WORKLOADS

    for key, spec in bench.SPECS.items():
        wl = WORKLOADS[key]()
        assert wl.name == spec["name"]
        assert (wl.shape.layers, wl.shape.kv_heads, wl.shape.head_dim) == (spec["layers"], spec["kv_heads"],
                                                                         spec["head_dim"])
        assert wl.queue.n == spec["n_req"] and int(wl.queue.context_tokens[0]) == spec["ctx"]
        assert float(wl.queue.cache_hit_ratio[0]) == spec["hit"] and int(wl.queue.query_tokens[0]) == spec["query"]
        nb = len(wl.slots[0])
        assert wl.pool_slots == spec["n_docs"] * nb
        shape, items, bt, num_pages, n_slots = bench.reference_sample(spec, 4)
        assert len(items) == spec["n_req"] * min(4, nb)
        assert shape.chunk_bytes == wl.shape.chunk_bytes
