#!/bin/bash
# ncu PCIe counters of the host-link ingest kernels (K1 zero-copy, K1b bulk; full heads and a TP8
# shard): pcie__read_bytes / pcie__throughput per launch.  gpurun --timeout 1200 -- 'bash tools/ncu_pcie.sh'
mkdir -p gpurun_out
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for t in ingest-zerocopy ingest-bulk ingest-tp8; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_ingest -c 40 --csv --log-file gpurun_out/ncu_pcie_$t.csv python tools/prof_targets.py $t > /dev/null 2>&1
  echo "$t rc=$?"
done
