"""Per CUDA source line: warp instructions and stall samples from an ncu
'--page source --csv --print-source cuda,sass' export. python tools/src_lines.py FILE [units] [min_frac]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
path = ""
hdr = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0] not in ("",):
        try:
            n = int(r[7]); smp = int(r[4])
        except ValueError:
            continue
        out.append((path, int(r[0]), n, smp, r[1][:100]))
T = sum(o[2] for o in out)
S = sum(o[3] for o in out)
print(f"total warp instructions {T:.0f} ({T / units:.0f} per unit), samples {S}")
for p, ln, n, smp, src in sorted(out, key=lambda o: (o[0], o[1])):
    if n > minf * T or smp > minf * S:
        print(f"{p:14s}{ln:5d} {n / units:8.0f} {100 * n / T:5.1f}% smp {100 * smp / S:5.1f}%  {src}")
