"""Stall samples / executed warp instructions per SOURCE line from an ncu source page:
   ncu -i rep --page source --csv --launch-skip K --launch-count 1 --print-source cuda,sass > x.csv
   python tools/src_hot.py x.csv [N]"""
import csv
import sys

N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, rows = None, None, []
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or not r[0].isdigit():
        continue
    m = r[len(r) - (len(hdr) - 4):]  # metric columns (the source text may hold commas)
    try:
        s, i = int(m[0] or 0), int(m[3] or 0)
    except ValueError:
        continue
    rows.append((fname, int(r[0]), s, i, r[1].strip()[:80]))
ts = sum(x[2] for x in rows) or 1
ti = sum(x[3] for x in rows) or 1
print(f"samples {ts}  warp instr {ti}")
for f, ln, s, i, src in sorted(rows, key=lambda x: -x[2])[:N]:
    print(f"{f}:{ln:<5d} {100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {src}")
