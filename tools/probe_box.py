"""Probe the GPU box: host RAM/CPU, topology, pinned H2D/D2H copy-engine bandwidth."""
import json, os, subprocess, time
import torch

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = os.cpu_count()
out["free"] = sh("free -g")
out["lscpu"] = sh("lscpu | head -30")
out["numa"] = sh("numactl -H 2>/dev/null || cat /sys/devices/system/node/online")
out["smi"] = sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current,memory.total,clocks.max.sm --format=csv")
out["topo"] = sh("nvidia-smi topo -m")
out["memlock"] = sh("ulimit -l")
out["shm"] = sh("df -h /dev/shm")
dev = torch.device("cuda:0")
torch.cuda.init()
res = {}
for mb in (4, 16, 64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best_h2d = best_d2h = 0.0
    for it in range(8):
        with torch.cuda.stream(s):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
        s.synchronize()
        best_h2d = max(best_h2d, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        with torch.cuda.stream(s):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
        s.synchronize()
        best_d2h = max(best_d2h, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    res[f"{mb}MB"] = {"h2d_GBps": round(best_h2d, 2), "d2h_GBps": round(best_d2h, 2)}
out["copy"] = res
# sustained H2D: 8 GiB streamed as 64 MB chunks back to back into a 4-slot ring
n = 64 << 20
hbuf = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
t0 = time.time(); hbuf.fill_(3); out["host_fill_8GiB_s"] = time.time() - t0
ring = torch.empty(4 * n, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for i in range((8 << 30) // n):
        ring[(i % 4) * n:(i % 4 + 1) * n].copy_(hbuf[i * n:(i + 1) * n], non_blocking=True)
    e1.record(s)
s.synchronize()
out["sustained_h2d_8GiB_64MB_chunks_GBps"] = (8 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
# bidirectional
d2 = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
h2 = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.time()
with torch.cuda.stream(s):
    d2.copy_(hbuf[: 1 << 30], non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(ring.repeat(4)[: 1 << 30], non_blocking=True)
torch.cuda.synchronize()
out["bidir_1GiB_each_s"] = time.time() - t0
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/probe_box.json", "w") as f:
    json.dump(out, f, indent=1)
