"""Per-CUDA-line warp-stall samples from an ncu report's source page (`--print-source cuda,sass`).

usage: python tools/ncu_cuda_lines.py <rep.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(r for r in rows if r and r[0] == "Line No")
    wi = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    data = []
    for r in rows:
        if len(r) > wi and r[0] and r[0] != "Line No" and r[0].isdigit():
            try:
                data.append((float(r[wi] or 0), float(r[ii] or 0), int(r[0]), r[1][:90]))
            except ValueError:
                pass
    tot = sum(d[0] for d in data) or 1
    toti = sum(d[1] for d in data) or 1
    print(f"total samples {tot:.0f}, warp instructions {toti:.0f}")
    for w, i, ln, s in sorted(data, reverse=True)[:top]:
        print(f"{w / tot * 100:5.1f}% stall  {i / toti * 100:5.1f}% inst  {ln:>5}  {s}")


if __name__ == "__main__":
    main()
