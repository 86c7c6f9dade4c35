"""Top SASS instructions by stall samples / executed count from an ncu source-page CSV.
   ncu -i rep --page source --csv --launch-skip K --launch-count 1 > x.csv; python tools/sass_hot.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[2].isdigit()]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
tot_i = sum(int(d["Instructions Executed"] or 0) for d in data)
print("total samples", tot_s, "total warp instr", tot_i)
for i, d in enumerate(data):
    d["idx"] = i
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:N]
for d in sorted(top, key=lambda d: d["idx"]):
    print(f'{d["idx"]:5d} {int(d["Warp Stall Sampling (All Samples)"]):8d} {100*int(d["Warp Stall Sampling (All Samples)"])/tot_s:5.1f}% {int(d["Instructions Executed"]):11d}  {d["Source"].strip()[:90]}')
