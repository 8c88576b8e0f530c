"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) of
`bench.py` into profiles/: the per-kernel launches of the C3 steps, each
kernel's share of the step, and profiles/ncu_traffic.json (read by bench.py for
roofline.traffic).

  python tools/launch_summary.py gpurun_out/launches.csv <first-id> <last-id> <out-prefix>
  (first-id -1: the last two steps of the list)

The ids select whole compress+decompress steps of the C3 tensor (n = 2^28)."""
import collections
import csv
import json
import sys

NAMES = {"tlc_absmax_kernel": "k1_absmax", "tlc_quant_qe_bulk_kernel": "k2_quant_qe",
         "tlc_quant_qe_kernel": "k2_quant_qe", "tlc_zre_kernel": "k3_zre",
         "tlc_zre_scan_kernel": "k4_zre_scan", "tlc_expand_dequant_kernel": "k5_expand_dequant"}


def main(path, lo, hi, prefix):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launch = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        d = launch.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    if lo < 0:                        # "auto": the last two COMPLETE C3 steps (K1 .. the K1 before the last K5)
        base = {i: d["name"].split("(")[0].split("::")[-1].split("<")[0] for i, d in launch.items()}
        hi = max(i for i, b in base.items() if b == "tlc_expand_dequant_kernel")
        lo = [i for i, b in base.items() if b == "tlc_absmax_kernel" and i < hi][-2]
    sel = [(i, d) for i, d in launch.items() if lo <= i <= hi]
    agg = collections.OrderedDict()
    out_rows = []
    for i, d in sel:
        base = d["name"].split("(")[0].split("::")[-1].split("<")[0]
        k = NAMES.get(base)
        if k is None:
            continue
        t, r_, w = d["gpu__time_duration.sum"], d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        out_rows.append((i, base, t, r_, w))
        a = agg.setdefault(k, {"launches": 0, "t": 0.0, "r": 0.0, "w": 0.0})
        a["t"] += t; a["r"] += r_; a["w"] += w
    steps = sum(1 for _, b, *_ in out_rows if b == "tlc_absmax_kernel")
    for a in agg.values():
        a["launches"] = steps
    total = sum(a["t"] for a in agg.values())
    with open(prefix + "_launches.csv", "w") as f:
        f.write("id,kernel,gpu_time_ns,dram_read_bytes,dram_write_bytes\n")
        for r in out_rows:
            f.write(",".join(str(x) for x in r) + "\n")
    traffic = {}
    lines = ["| kernel | ns per step | share of step | DRAM read / write per step (bytes) |", "|---|---|---|---|"]
    for k, a in agg.items():
        lines.append(f"| {k} | {a['t'] / steps:.0f} | {a['t'] / total:.3f} | {a['r'] / steps:.0f} / {a['w'] / steps:.0f} |")
        traffic[k] = {"n": 1 << 28, "dram_bytes_per_launch": (a["r"] + a["w"]) / steps, "dram_read": a["r"] / steps,
                      "dram_write": a["w"] / steps, "gpu_time_ns": a["t"] / steps,
                      "source": f"{prefix}_launches.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                                f"dram__bytes_write.sum --cache-control none --clock-control none; launches {lo}-{hi})"}
    with open(prefix + "_launch_summary.md", "w") as f:
        f.write(f"Launch list of {steps} C3 steps (ids {lo}-{hi}), serialised under ncu, caches not flushed.\n\n")
        f.write("\n".join(lines) + "\n")
    json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
