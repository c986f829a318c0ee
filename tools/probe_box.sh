#!/bin/bash
# One-off box probe: host cores/RAM, GPU topology, toolchain sanity.
set -x
nproc; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"
free -g; cat /proc/cpuinfo | grep "model name" | head -1
nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import torch, time
print(torch.cuda.device_count(), torch.cuda.get_device_name(0), torch.cuda.mem_get_info())
p = torch.cuda.get_device_properties(0); print(p)
# pinned H2D bandwidth
x = torch.empty(1<<30, dtype=torch.uint8).pin_memory(); y = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt=time.perf_counter()-t; print('H2D GB/s', 5*(1<<30)/dt/1e9)
t=time.perf_counter()
for _ in range(5): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); dt=time.perf_counter()-t; print('D2H GB/s', 5*(1<<30)/dt/1e9)
t=time.perf_counter(); z = torch.empty(8<<30, dtype=torch.uint8).pin_memory(); print('pin 8GB s', time.perf_counter()-t)
PY
