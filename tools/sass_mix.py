"""Opcode mix and stall samples of an ncu source page (--page source --csv --print-source sass)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter()
stall = collections.Counter()
seq = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = int(r[ix["Instructions Executed"]] or 0)
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot[op.split(".")[0]] += n
    stall[op.split(".")[0]] += smp
    seq.append((r[ix["Address"]], src, n, smp))
T = sum(tot.values())
S = sum(stall.values())
print(f"total warp instructions {T}, stall samples {S}")
for op, n in tot.most_common(30):
    print(f"{op:12s} {n:12d} {100 * n / T:5.1f}%   samples {100 * stall[op] / max(S, 1):5.1f}%")
if len(sys.argv) > 2:  # dump the hottest instructions by samples
    for a, src, n, smp in sorted(seq, key=lambda x: -x[3])[: int(sys.argv[2])]:
        print(f"{a[-5:]} {smp:6d} {n:9d}  {src[:90]}")
