"""Summarise an ncu --set full report of one c2 update (+ optional launch list) into
profiles/: <name>_ncu.json (per-kernel metrics; summed DRAM bytes of the classify
kernels, the 'traffic' bench.py reports) and <name>_launches.csv (copy).
usage: python tools/ncu_summary.py REPORT.ncu-rep NAME [LAUNCHES.csv]"""
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
        "grid": "launch__grid_size", "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"}
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
cls = [k for k in kernels if any(s in k["kernel"] for s in ("touch_warp", "narrow_kernel", "apply_warp"))]
rd = sum(k.get("dram_read_bytes", 0) for k in cls)
wr = sum(k.get("dram_write_bytes", 0) for k in cls)
out = {"source": f"ncu --set full --clock-control none, one c2 update (tools/step_once.py), {rep.split('/')[-1]}",
       "kernels": kernels, "dram__bytes_read.sum": [str(rd), "byte"], "dram__bytes_write.sum": [str(wr), "byte"],
       "classify_duration_us": sum(k.get("duration_us", 0) for k in cls),
       "note": "ncu flushes caches before each kernel: the narrow kernel's operands that touch prefetched into L2 "
               "are re-read cold here, so the summed DRAM bytes overstate a live update's traffic"}
json.dump(out, open(f"profiles/{name}_ncu.json", "w"), indent=1)
if len(sys.argv) > 3:
    shutil.copy(sys.argv[3], f"profiles/{name}_launches.csv")
for k in kernels:
    print(f"{k['kernel'][:40]:40s} {k.get('duration_us', 0):7.2f} us  dram {k.get('dram_read_bytes', 0) / 1e6:6.2f} MB  "
          f"warps {k.get('warps_active_pct', 0):5.1f}%  issue {k.get('issue_active_pct', 0):5.1f}%  regs {k.get('registers')}")
print("classify dram MB", rd / 1e6, wr / 1e6)
