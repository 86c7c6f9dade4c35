"""Executed warp instructions and stall samples grouped by kernel role (line ranges
given on the command line) from an ncu source page (--print-source cuda,sass csv).
   python tools/src_roles.py x.csv nrows file:lo-hi=role ..."""
import csv
import sys


def parse(path):
    hdr, fname, out = None, None, []
    with open(path, encoding="utf-8", errors="replace") as fh:
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
                continue
            m = r[len(r) - (len(hdr) - 4):]
            names = hdr[4:]
            col = {h: k for k, h in enumerate(names)}
            try:
                s = int(m[col["Warp Stall Sampling (All Samples)"]] or 0)
                i = int(m[col["Instructions Executed"]] or 0)
            except (ValueError, IndexError):
                continue
            out.append((fname, int(r[0]), s, i))
    return out


def main():
    rows = parse(sys.argv[1])
    nrows = float(sys.argv[2])
    spec = []
    for a in sys.argv[3:]:
        rng, role = a.split("=")
        f, lh = rng.split(":")
        lo, hi = lh.split("-")
        spec.append((f, int(lo), int(hi), role))
    agg = {}
    for f, ln, s, i in rows:
        role = next((ro for (ff, lo, hi, ro) in spec if ff == f and lo <= ln <= hi), f + " other")
        a = agg.setdefault(role, [0, 0])
        a[0] += s
        a[1] += i
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instr {ti:.3e} ({ti / nrows:.0f} per row), samples {ts}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:24s} smp {100 * v[0] / ts:5.1f}%  ins {100 * v[1] / ti:5.1f}%  per-row {v[1] / nrows:7.0f}")


if __name__ == "__main__":
    main()
