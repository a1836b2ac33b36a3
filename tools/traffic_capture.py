"""DRAM traffic of one fused lars_step launch, measured with ncu on the
current build (the bench's roofline `traffic`).

Runs `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum` on tools/profile_step.py (same workload and shard
plan as the bench, carried ||w||; ncu flushes the caches before the
profiled launch, like the bench's L2 flush) and returns the per-launch
bytes.  Bench numbers are never taken from this run: only byte counts.

    python tools/traffic_capture.py [--workload resnet50] [--world 1 --rank 0]
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def under_profiler():
    return bool(os.environ.get("CUDA_INJECTION64_PATH") or os.environ.get("NV_COMPUTE_PROFILER_PERFWORKS_DIR"))


def capture(workload="resnet50", world=1, rank=0, timeout=240):
    """{'read': B, 'write': B, 'duration_ns': t} per launch, or {'error': ...}."""
    if under_profiler():
        return {"error": "already running under a profiler"}
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    cmd = [ncu, "--metrics", METRICS, "--clock-control", "none", "-k", "regex:lars_step_kernel",
           "--launch-skip", "3", "--launch-count", "1", "--csv",
           sys.executable, os.path.join(HERE, "tools", "profile_step.py"), "--workload", workload,
           "--steps", "5", "--world", str(world), "--rank", str(rank)]
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=HERE)
    except subprocess.TimeoutExpired:
        return {"error": f"ncu timed out after {timeout} s"}
    rows = [r for r in csv.reader(io.StringIO(p.stdout)) if r]
    hdr = next((r for r in rows if "Metric Name" in r), None)
    if hdr is None:
        return {"error": f"ncu rc={p.returncode}: {(p.stderr or p.stdout)[-300:]}"}
    i_name, i_unit, i_val = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}
    out = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_val:
            continue
        v = float(r[i_val].replace(",", "")) * scale.get(r[i_unit], 1)
        key = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write",
               "gpu__time_duration.sum": "duration_ns"}.get(r[i_name])
        if key:
            out[key] = int(round(v))
    if "read" not in out or "write" not in out:
        return {"error": "dram metrics missing from the ncu output"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    a = ap.parse_args()
    print(json.dumps(capture(a.workload, a.world, a.rank)))


if __name__ == "__main__":
    main()
