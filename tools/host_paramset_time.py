"""Wall time of optim.apply_update on a reference-style fp64 ParamSet (the
stock batchlab.nn.ParamSet when installed) for several pipeline part sizes.

    python tools/host_paramset_time.py [--workload resnet50] [--parts-min 1e12,4194304,1048576]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1709_05011_b200 import hostset, layouts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="resnet50")
ap.add_argument("--parts-min", default="1000000000000,4194304,2097152")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
layout = layouts.get(args.workload)
for pm in [int(float(x)) for x in args.parts_min.split(",")]:
    hostset.PART_MIN_ELEMS = pm
    out = bench.e2e_host_paramset(layout, args.steps, None)
    print(f"PART_MIN_ELEMS {pm:>14d}: {out['ms_per_step']:8.3f} ms  ({out['value']} GB/s)", flush=True)
