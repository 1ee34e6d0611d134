"""Summarise an ncu --set full report of one update (+ optional launch list) into
profiles/: <name>_ncu.json (per-kernel metrics incl. FP32/FP64 pipe utilisation; the
summed DRAM bytes of one update's kernels, the 'traffic' bench.py reports) and
<name>_launches.csv (copy).
usage: python tools/ncu_summary.py REPORT.ncu-rep NAME [LAUNCHES.csv] [SOURCE-DESCRIPTION]"""
import csv
import io
import json
import shutil
import subprocess
import sys

rep, name = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
keys = {"duration_us": "gpu__time_duration.sum", "dram_read_bytes": "dram__bytes_read.sum",
        "dram_write_bytes": "dram__bytes_write.sum", "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct", "registers": "launch__registers_per_thread",
        "grid": "launch__grid_size", "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "fp32_inst_pipe_fma": "sm__inst_executed_pipe_fma.sum", "warp_inst": "smsp__inst_executed.sum",
        "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio"}
kernels = []
for row in rows[2:]:
    k = {"kernel": row[h.index("Kernel Name")]}
    for out, m in keys.items():
        if m not in h:
            continue
        v, u = row[h.index(m)], units[h.index(m)]
        try:
            k[out] = float(v.replace(",", "")) * scale.get(u, 1)
        except ValueError:
            k[out] = v
    kernels.append(k)
upd = ("pose_kernel", "bin_scatter", "bin_cells", "bin_small", "cells_touch", "touch_warp_kernel<0", "touch_warp_kernel<false", "narrow_kernel<0",
       "narrow_kernel<false", "touch_cta", "narrow_over", "narrow_under", "single_cells", "apply_warp", "gray_count", "gray_write")
seen, cls = set(), []
for k in kernels:  # one launch of each update kernel
    tag = next((t for t in upd if t in k["kernel"]), None)
    if tag and tag not in seen:
        seen.add(tag)
        cls.append(k)
rd = sum(k.get("dram_read_bytes", 0) for k in cls)
wr = sum(k.get("dram_write_bytes", 0) for k in cls)
src = sys.argv[4] if len(sys.argv) > 4 else "one update (tools/step_once.py)"
out = {"source": f"ncu --set full --clock-control none, {src}, {rep.split('/')[-1]}",
       "kernels": kernels, "update_kernels": [k["kernel"] for k in cls],
       "dram__bytes_read.sum": [str(rd), "byte"], "dram__bytes_write.sum": [str(wr), "byte"],
       "dram_bytes_per_update": rd + wr, "update_duration_us": sum(k.get("duration_us", 0) for k in cls),
       "note": "ncu flushes caches before each kernel and serialises them: durations are cold-cache, and "
               "operands a kernel reads that its predecessor left in L2 are re-read from DRAM here"}
json.dump(out, open(f"profiles/{name}_ncu.json", "w"), indent=1)
if len(sys.argv) > 3 and sys.argv[3]:
    shutil.copy(sys.argv[3], f"profiles/{name}_launches.csv")
for k in kernels:
    print(f"{k['kernel'][:40]:40s} {k.get('duration_us', 0):7.2f} us  dram {k.get('dram_read_bytes', 0) / 1e6:6.2f} MB  "
          f"warps {k.get('warps_active_pct', 0):5.1f}%  issue {k.get('issue_active_pct', 0):5.1f}%  regs {k.get('registers')}")
print("update dram MB", rd / 1e6, wr / 1e6, "kernels", [k["kernel"][:30] for k in cls])
