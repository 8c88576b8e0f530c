"""Per-source-line totals of an ncu SASS source page.

usage: python tools/ncu_lines.py <ncu-source.csv> <cubin> <mangled-kernel> [top] [--outer]
(--outer attributes inlined code to its outermost call site)

The csv is `ncu -i rep --page source --csv --kernel-name K` (SASS view, one row
per instruction in address order); the cubin's `nvdisasm -g` line comments map
each instruction offset (16 bytes per instruction) to file:line.
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn, outer=False):
    out = subprocess.run(["nvdisasm", "-gi" if outer else "-g", "-c", cubin], capture_output=True,
                         text=True).stdout
    sec = False
    cur = "?"
    m = {}
    for ln in out.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            sec = (".text." + fn + " ") in ln + " "
            continue
        if not sec:
            continue
        g = re.findall(r'"([^"]*)", line (\d+)', ln) if ln.lstrip().startswith("//##") else None
        if g:
            f, l = g[-1] if outer else g[0]      # outermost call site, or the innermost line
            cur = f.split("/")[-1] + ":" + l
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    args = [a for a in sys.argv[1:] if a != "--outer"]
    outer = "--outer" in sys.argv
    path, cubin, fn = args[:3]
    top = int(args[3]) if len(args) > 3 else 40
    rows = list(csv.reader(open(path)))
    h = rows[1]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    ss = h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ie]
    lm = line_map(cubin, fn, outer)
    inst = collections.Counter()
    samp = collections.Counter()
    data = [r for r in data if r[ie].strip().isdigit() or r[ie].strip() == ""]   # repeated header rows
    for i, r in enumerate(data):
        key = lm.get(16 * i, "?")
        inst[key] += int(r[ie] or 0)
        samp[key] += int(r[ss] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total warp-instr {ti}, stall samples {ts}")
    for k, v in inst.most_common(top):
        print(f"{k:28s} inst {v:10d} ({100*v/ti:5.1f}%)  samples {samp[k]:6d} ({100*samp[k]/max(ts,1):5.1f}%)")


if __name__ == "__main__":
    main()
