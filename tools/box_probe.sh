#!/bin/bash
# P0 box probe: host facts that set the roofline denominators and memory feasibility.
out=gpurun_out/box_probe.txt
{
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== meminfo"; head -5 /proc/meminfo
echo "== numactl"; (numactl -H 2>/dev/null || echo "no numactl"; ls /sys/devices/system/node/ )
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi -q | grep -iA6 "PCI$\|Link Width\|Generation" | head -40
echo "== ulimit -l"; ulimit -l
} > $out 2>&1
python - >> $out 2>&1 <<'PY'
import torch, time
print("torch", torch.__version__, torch.cuda.get_device_name(0))
p = torch.cuda.get_device_properties(0); print(p)
# pinned H2D probe
for gib in (1,):
    n = gib << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("H2D pinned GB/s", 5*n/ (s.elapsed_time(e)*1e-3) / 1e9)
    s.record();
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("D2H pinned GB/s", 5*n/ (s.elapsed_time(e)*1e-3) / 1e9)
# big pin test: how long to pin 16 GiB
t=time.time(); x = torch.empty(16<<30, dtype=torch.uint8, pin_memory=True); print("pin 16GiB s", time.time()-t); del x
PY
