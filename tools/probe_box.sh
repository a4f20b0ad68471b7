#!/bin/bash
# One-off environment probe of a GPU box (host cores/RAM, device properties).
set -x
nproc; cat /proc/cpuinfo | grep 'model name' | head -1; free -g; lscpu | head -20
nvidia-smi
python - <<'PY'
import torch, os
p = torch.cuda.get_device_properties(0)
print(p)
print("sms", p.multi_processor_count, "l2", getattr(p, "L2_cache_size", None), "mem", p.total_memory)
print("affinity", len(os.sched_getaffinity(0)))
f, t = torch.cuda.mem_get_info(); print("free", f, "total", t)
PY
