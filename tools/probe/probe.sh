#!/bin/bash
set -x
mkdir -p gpurun_out
{
nproc; lscpu | head -30; free -g; ulimit -l; cat /sys/fs/cgroup/memory.max 2>/dev/null
nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -iA3 "PCIe Generation\|Link Width" | head -30
numactl --hardware 2>/dev/null
timeout 300 ./tools/probe/hostlink_probe 4096
python -c "import torch,time; t=time.time(); x=torch.empty(64<<30,dtype=torch.uint8,pin_memory=True); print('pin64G s',time.time()-t)"
} > gpurun_out/probe.txt 2>&1
