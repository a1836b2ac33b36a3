"""Summarise an .ncu-rep: key raw metrics + top stall reasons / SASS lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N]
"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 12
    rows = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[hdr.index("Kernel Name")][:90])
        for w in WANT:
            if w in hdr:
                print(f"  {w:60s} {r[hdr.index(w)]:>16s} {units[hdr.index(w)]}")
    src = list(csv.reader(ncu(rep, "--page", "source", "--csv", "--print-source=sass").splitlines()))
    if len(src) < 3:
        return
    h = src[1]
    idx = h.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    data = [r for r in src[2:] if len(r) >= len(h) - 1]
    tot = sum(int(r[idx] or 0) for r in data)
    agg = {}
    for r in data:
        for i in cols:
            agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
    print(f"  stall samples {tot}: " + ", ".join(f"{k[6:]} {100 * v / tot:.1f}%"
                                               for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    top = sorted(data, key=lambda r: -int(r[idx] or 0))[:nsass]
    for r in top:
        print(f"    {100 * int(r[idx]) / tot:5.1f}%  {r[1].strip()[:70]}")


if __name__ == "__main__":
    main()
