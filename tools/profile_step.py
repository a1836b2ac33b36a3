"""Run a few LARS steps on one GPU for ncu (no timing, no graph).

    python tools/profile_step.py [--workload resnet50] [--steps 6] [--no-carry] [--split]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1709_05011_b200 import layouts, optim  # noqa: E402
from paper_1709_05011_b200.cluster import DataParallelLars  # noqa: E402
from paper_1709_05011_b200.flat import FlatParamSet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--no-carry", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    layout = layouts.get(args.workload)
    params = FlatParamSet(layout, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for grp in params:
        if grp.category == "weight":
            grp.param.uniform_(-0.05, 0.05, generator=g)
        elif grp.category == "norm-scale":
            grp.param.fill_(1.0)
        grp.grad.normal_(0, 1.0, generator=g)
    hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5,
                           lars_enabled=True)
    st = optim.ScheduleState(3515, 39)
    dp = DataParallelLars(params)
    flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    clean = torch.ones(1 << 26, dtype=torch.float32, device=dev)
    for _ in range(args.steps):
        flush.zero_()
        clean.sum()
        if args.no_carry:
            params.invalidate_norm_cache()
        dp.step(hp, st, grad_scale=1.0 / 32768)
    torch.cuda.synchronize()
    print("ok", optim.step_info(params))


if __name__ == "__main__":
    main()
