"""Summarise an ncu --set full report: one row per kernel of the headline
metrics, the full details page, the source-level stall page of the first
kernel, and the per-pass DRAM traffic JSON that bench.py reports as
roofline.traffic (with the plan it was captured on; bench.py uses it only
when the plan matches).

    python tools/ncu_summary.py gpurun_out/prof_n32.ncu-rep gpurun_out/r02_n32 32
      -> gpurun_out/r02_n32_summary.csv, _details.csv, _source.csv, _traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__cluster_dim_x", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed"]
idx = {h: i for i, h in enumerate(head)}
cols = [w for w in want if w in idx]
with open(f"{prefix}_summary.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["Kernel Name"] + cols)
    w.writerow([""] + [units[idx[c]] for c in cols])
    for r in data:
        w.writerow([r[idx["Kernel Name"]]] + [r[idx[c]] for c in cols])
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True, check=True).stdout
with open(f"{prefix}_details.csv", "w") as f:
    f.write(det)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
with open(f"{prefix}_source.csv", "w") as f:
    f.write(src)


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(v.replace(",", "")) * scale


passes = []
data = [r for r in data if "k32_sample" not in r[idx["Kernel Name"]]]  # the one-CTA sample test is not a pass
for i, r in enumerate(data):
    passes.append({"pass": i, "kernel": r[idx["Kernel Name"]].split("(")[0].replace("void ", ""),
                   "duration_ms": float(r[idx["gpu__time_duration.sum"]].replace(",", "")) *
                   {"ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ns": 1e-6, "nsecond": 1e-6}.get(
                       units[idx["gpu__time_duration.sum"]], 1),
                   "dram_read_bytes": to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]),
                   "dram_write_bytes": to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])})
plan = None
alg = 16 * 2 ** n
compact = any("k32_" in p["kernel"] for p in passes)  # the compact plan's int32-engine kernels
try:
    import ctypes
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1607_01039_b200 import _lib, sharded

    if compact:  # the plan key bench.py compares with: [["compact", k, r, engine], ...]
        L = _lib.lib()
        plan, alg = [], []
        for i in range(L.bw_compact_npasses(n)):
            k_, r_, e_, b_ = (ctypes.c_int(0) for _ in range(4))
            _lib.check(L.bw_compact_pass_info(n, i, ctypes.byref(k_), ctypes.byref(r_), ctypes.byref(e_), ctypes.byref(b_)))
            plan.append(["compact", k_.value, r_.value, e_.value])
            alg.append(b_.value * 2 ** n)
    else:
        plan = [[q["kind"], q["k"], q["r"], q.get("split_a", 0), q.get("k2", 0)] for q in sharded.plan(n, 0)["passes"]]
except Exception as e:  # noqa: BLE001 -- the summary is still useful without the plan
    print("plan unavailable:", e)
with open(f"{prefix}_traffic.json", "w") as f:
    json.dump({"source": f"ncu --set full --clock-control none ({rep})", "n": n, "plan": plan,
               "algorithmic_bytes_per_pass": alg, "passes": passes}, f, indent=1)
for p in passes:
    print(p)
