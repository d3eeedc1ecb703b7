"""Per-CUDA-source-line hot spots of an ncu report (dev tool).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [top_n]

Reads `ncu --page source --print-source cuda,sass` and prints the source lines
with the most warp-stall samples and executed warp instructions (inlined
helpers are attributed to their own lines).
"""
import csv
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = "?"
    res = []
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] and r[0].isdigit() and len(r) > 7 and r[4] not in ("-", ""):
            try:
                res.append((fname, int(r[0]), r[1].strip(), float(r[4] or 0), float(r[7] or 0)))
            except ValueError:  # source text with unbalanced quotes (inline asm)
                continue
    return res


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    res = lines(rep)
    ts = sum(x[3] for x in res) or 1
    ti = sum(x[4] for x in res) or 1
    print(f"{'file:line':28s} {'stall%':>7s} {'inst%':>7s}  source")
    for f, ln, src, s, i in sorted(res, key=lambda x: -x[3])[:n]:
        print(f"{f + ':' + str(ln):28s} {s / ts * 100:7.2f} {i / ti * 100:7.2f}  {src[:90]}")


if __name__ == "__main__":
    main()
