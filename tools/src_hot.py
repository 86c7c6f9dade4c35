"""Stall samples / executed warp instructions per SOURCE line from an ncu source page:
   ncu -i rep --page source --csv --launch-skip K --launch-count 1 --print-source cuda,sass > x.csv
   python tools/src_hot.py x.csv [N] [--by ins|smp]"""
import csv
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
N = int(args[1]) if len(args) > 1 else 40
by = "ins" if "--by" in sys.argv and sys.argv[sys.argv.index("--by") + 1] == "ins" else "smp"
fname, hdr, rows = None, None, []
with open(args[0], encoding="utf-8", errors="replace") as fh:
    for r in csv.reader(fh):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue  # SASS rows (empty line number) are already summed into their source line
        col = {h: k for k, h in enumerate(hdr)}
        try:
            s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
            i = int(r[col["Instructions Executed"]] or 0)
        except (KeyError, ValueError, IndexError):
            continue
        rows.append((fname, int(r[0]), s, i, r[1].strip()[:80]))
ts = sum(x[2] for x in rows) or 1
ti = sum(x[3] for x in rows) or 1
print(f"samples {ts}  warp instr {ti}")
key = (lambda x: -x[3]) if by == "ins" else (lambda x: -x[2])
for f, ln, s, i, src in sorted(rows, key=key)[:N]:
    print(f"{f}:{ln:<5d} {100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {src}")
