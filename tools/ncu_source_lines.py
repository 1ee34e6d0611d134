"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export to per-source-line
warp-stall samples with the dominant stall reasons (profiling helper, not product code)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if len(r) > 10 and r[0] == "Line No")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
out, fname, tot_by = [], None, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        try:
            w = int(r[4])
        except ValueError:
            continue
        rs = sorted(((int(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:3]
        for v, h in rs:
            tot_by[h] = tot_by.get(h, 0) + v
        out.append((w, fname, int(r[0]), r[1].strip()[:90], rs))
tot = sum(o[0] for o in out) or 1
print("total samples", tot, "| by reason:", sorted(tot_by.items(), key=lambda x: -x[1])[:8])
for w, f, ln, src, rs in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{w:6d} {100 * w / tot:5.1f}% {f}:{ln:<4d} {src:90s} {' '.join(f'{h}={v}' for v, h in rs if v)}")
