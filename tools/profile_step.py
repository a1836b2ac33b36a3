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
    ap.add_argument("--world", type=int, default=1,
                    help="profile the single-GPU fused kernel on rank --rank's shard plan")
    ap.add_argument("--rank", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    layout = layouts.get(args.workload)
    params = FlatParamSet(layout, dev, world_size=args.world, rank=args.rank)
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
    flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    clean = torch.ones(1 << 26, dtype=torch.float32, device=dev)
    if args.world == 1:
        dp = DataParallelLars(params)
        step = lambda i: dp.step(hp, st, grad_scale=1.0 / 32768)  # noqa: E731
    else:
        from paper_1709_05011_b200 import _native as nat
        from paper_1709_05011_b200.flat import _ptr, _stream
        eng = params.engine()
        plan, ws = eng.plan(frozenset(hp.lars_skip_categories))

        def step(i):
            flags = nat.LARS_STEP_USE_WCARRY if i > 0 and not args.no_carry else 0
            h = optim.native_hparams(hp, st, lr=0.01, grad_scale=1.0 / 32768, flags=flags)
            nat.check(nat.load().lars_step(
                plan.handle, _ptr(params.param_shard), _ptr(params.grad_shard_of_full),
                _ptr(params.momentum), nat.ctypes.byref(h), _ptr(eng.d_iter), _ptr(eng.d_sumsq),
                _ptr(eng.d_lambda), _ptr(eng.d_info), _ptr(ws), _stream()))
    for i in range(args.steps):
        flush.zero_()
        clean.sum()
        if args.no_carry:
            params.invalidate_norm_cache()
        step(i)
    torch.cuda.synchronize()
    print("ok", optim.step_info(params))


if __name__ == "__main__":
    main()
