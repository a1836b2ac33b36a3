"""Top stalled CUDA source lines of an .ncu-rep (needs -lineinfo): sums the
SASS-level warp-stall samples of each source line.

    python tools/ncu_lines.py report.ncu-rep [--top 20]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    per, src, cur = {}, {}, None
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_s:
            continue
        if r[0]:
            cur = r[0]
            src[cur] = r[1].strip()
            continue
        try:
            per[cur] = per.get(cur, 0) + float(r[i_s] or 0)
        except ValueError:
            pass
    tot = sum(per.values()) or 1
    for ln, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  L{ln:>5}  {src.get(ln, '')[:110]}")


if __name__ == "__main__":
    main()
