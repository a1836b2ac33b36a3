"""Markdown table from the bench lines of tools/config_sweep.sh.

    python tools/config_sweep_table.py gpurun_out/sweep > profiles/r01_config_sweep.md
"""
import glob
import json
import os
import sys


def main():
    rows = []
    for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        c, r = d["config"], d["roofline"]
        sd = d.get("scaling_defs") or {}
        rows.append((c["params"], d["n_gpus"], c["workload"].split(" ")[0], c["layers"], d["ms_per_step"] * 1e3,
                     d["value"], r["kernel_us"], r["frac"], sd.get("kernel_only_strong_eff"),
                     sd.get("step_roofline_eff"), sd.get("nvlink_gbs_per_direction"), d["backend"],
                     d["e2e"]["value"]))
    rows.sort()
    print("| workload | params | layers | GPUs | step µs | value GB/s (20 B/param, whole job) | "
          "kernel µs | HBM frac (N=1) | E_k | E_s | NVLink GB/s/dir | backend | e2e GB/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p, n, w, L, us, v, k, fr, ek, es, nv, be, e2e in rows:
        f = lambda x, fmt: "—" if x is None else fmt.format(x)  # noqa: E731
        print(f"| {w} | {p:,} | {L} | {n} | {us:.1f} | {v:.0f} | {k:.1f} | "
              f"{f(fr if n == 1 else None, '{:.3f}')} | {f(ek, '{:.2f}')} | {f(es, '{:.2f}')} | "
              f"{f(nv, '{:.0f}')} | {be} | {e2e:.0f} |")


if __name__ == "__main__":
    main()
