"""One markdown table row per kernel of ncu reports (`ncu -i <rep> --page details --csv`):
duration, DRAM throughput and bytes, issue-slot use, executed warp instructions, occupancy,
registers.  usage: python tools/ncu_summary.py gpurun_out/a.ncu-rep [...]"""
import csv
import io
import os
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Instructions",
        "Achieved Occupancy", "Registers Per Thread", "Grid Size"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if not r:
        return []
    h = r[0]
    ki, ii, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    ker = {}
    for x in r[1:]:
        d = ker.setdefault(x[ii], {"name": x[ki].split("(")[0].replace("void ", "")})
        if x[mi] in WANT and (x[mi] not in d or x[mi] != "Memory Throughput" or "byte" in x[ui].lower()):
            d[x[mi] + (" [" + x[ui] + "]" if x[ui] else "")] = x[vi]
    return list(ker.values())


def main():
    print("| report | kernel | " + " | ".join(WANT) + " |")
    print("|" + "---|" * (len(WANT) + 2))
    for rep in sys.argv[1:]:
        for d in rows(rep):
            vals = []
            for w in WANT:
                k = next((k for k in d if k.startswith(w)), None)
                vals.append(f"{d[k]} {k[len(w):].strip(' []')}".strip() if k else "")
            print(f"| {os.path.basename(rep).replace('.ncu-rep', '')} | {d['name']} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
