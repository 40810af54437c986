"""Summarise ncu reports (--set full captures) into one JSON line per launch.

python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] > profiles/rNN_ncu_x.jsonl
Fields: kernel, grid, duration, DRAM bytes read/written (the roofline's `traffic`),
DRAM / SM / tensor-pipe utilisation and registers, straight from ncu's raw page."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "kernel": "Kernel Name", "grid": "Grid Size", "block": "Block Size",
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
}
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    for row in r[2:]:
        rec = {"report": path.split("/")[-1]}
        for k, name in KEYS.items():
            if name not in head:
                continue
            i = head.index(name)
            v, u = row[i], units[i]
            try:
                f = float(v.replace(",", ""))
                if k.endswith("_bytes"):
                    f *= SCALE.get(u, 1.0)
                elif k == "duration_us":
                    f *= SCALE.get(u, 1.0)
                rec[k] = round(f, 3)
            except ValueError:
                rec[k] = v
        if "dram_read_bytes" in rec and "dram_write_bytes" in rec:
            rec["traffic_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        yield rec


for p in sys.argv[1:]:
    for rec in rows(p):
        print(json.dumps(rec))
