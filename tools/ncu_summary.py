"""Summarise ncu outputs into profiles/ (run here, after gpurun brings them back).

  python tools/ncu_summary.py launches gpurun_out/launches_r1.csv > profiles/r1_launches.md
  python tools/ncu_summary.py report gpurun_out/prof.ncu-rep     > profiles/r1_<kernel>.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L2 Hit Rate", "L1/TEX Hit Rate", "Registers Per Thread",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct",
       "l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
       "gpu__time_duration.sum"]


def launches(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"])
        unit = r.get("Metric Unit", "")
        if unit in ("nsecond", "ns"):
            v /= 1e3
        elif unit in ("msecond", "ms"):
            v *= 1e3
        per.setdefault(name, []).append(v)
    total = sum(sum(v) for v in per.values())
    print(f"# Launch list ({path})\n")
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised; compare shares)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---:|---:|---:|---:|")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{name}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.1f} | {sum(v)/total:.1%} |")
    print(f"\nTotal device time: {total/1e3:.2f} ms over {sum(len(v) for v in per.values())} launches")


def report(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.DictReader(io.StringIO(det)))
    by_id = collections.OrderedDict()
    for r in rows:
        by_id.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = (
            r["Metric Value"], r["Metric Unit"])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rr[0], rr[1], rr[2:]
    print(f"# ncu --set full summary ({path})\n")
    for k, (kid, d) in enumerate(by_id.items()):
        print(f"## launch {kid}: `{d['name'][:120]}`\n")
        print("| metric | value |")
        print("|---|---|")
        for key in KEYS:
            if key in d:
                print(f"| {key} | {d[key][0]} {d[key][1]} |")
        if k < len(vals):
            for key in RAW:
                # raw-page columns may carry a section prefix ("TPC.TriageCompute.<metric>")
                i = next((j for j, h in enumerate(hdr) if h == key or h.endswith("." + key)), None)
                if i is not None:
                    print(f"| {key} | {vals[k][i]} {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
