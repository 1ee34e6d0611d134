"""Per-kernel mean durations (us) from an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[r[ui]]
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    d[name].append(v)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 1
print(" | ".join(f"{k[-22:]} {sum(v[skip:]) / max(1, len(v[skip:])):.1f}" for k, v in d.items() if any(s in k for s in ("pose", "bin", "touch", "narrow", "apply", "gray"))))
