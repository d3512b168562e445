"""Stall samples and instructions per barrier-delimited region of an ncu SASS source page, plus the
top stall reasons (raw page). python tools/ncu_regions.py TAG  (reads gpurun_out/TAG_{sass,raw}.csv)"""
import csv
import sys

tag = sys.argv[1]
nblk = float(sys.argv[2]) if len(sys.argv) > 2 else 4096.0
rows = list(csv.reader(open(f"{tag}_raw.csv")))
d = dict(zip(rows[0], rows[2]))
st = {k: float(v.replace(",", "")) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
tot = sum(st.values())
print("  ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
for k in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    print(k, d.get(k))
rows = list(csv.reader(open(f"{tag}_sass.csv")))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seq = [(r[ix["Address"]][-5:], r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
        int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in rows[2:] if len(r) >= len(hdr)]
tot = sum(x[3] for x in seq)
cur = ins = 0
start = seq[0][0]
for i, (a, src, n, smp) in enumerate(seq):
    cur += smp
    ins += n
    if "BAR.SYNC" in src or "EXIT" in src or i == len(seq) - 1:
        if ins:
            print(f"{start}-{a}  samples {100 * cur / tot:5.1f}%  warp-instr/CTA {ins / nblk:8.0f}  ends: {src[:50]}")
        cur = ins = 0
        start = a
