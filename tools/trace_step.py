"""Per-warp phase timeline of the fused LARS step (profiling build).

    python -m paper_1709_05011_b200.build --trace
    LARS_B200_LIB=liblars_b200_trace.so python tools/trace_step.py [--workload resnet50]

Prints, over all warps, the distribution of: phase A (norms) duration, wait at
the grid barrier, coefficient setup, phase B (update) duration, and the
kernel span.  Timestamps are %globaltimer (ns).
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LARS_B200_LIB", "liblars_b200_trace.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1709_05011_b200 import _native as nat, layouts, optim  # noqa: E402
from paper_1709_05011_b200.cluster import DataParallelLars  # noqa: E402
from paper_1709_05011_b200.flat import FlatParamSet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-carry", action="store_true")
    ap.add_argument("--world", type=int, default=1, help="trace rank --rank's shard plan of a world")
    ap.add_argument("--rank", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    layout = layouts.get(args.workload)
    params = FlatParamSet(layout, dev, world_size=args.world, rank=args.rank)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for grp in params:
        grp.param.uniform_(-0.05, 0.05, generator=g)
        grp.grad.normal_(0, 1.0, generator=g)
    hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5,
                           lars_enabled=True)
    st = optim.ScheduleState(3515, 39)
    eng = params.engine()
    key = frozenset(hp.lars_skip_categories)
    plan, ws = eng.plan(key)
    lib = nat.load()
    from paper_1709_05011_b200.flat import _ptr, _stream
    flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    clean = torch.ones(1 << 26, dtype=torch.float32, device=dev)
    ev = []
    for i in range(args.steps):
        flush.zero_()
        clean.sum()
        flags = nat.LARS_STEP_USE_WCARRY if (i > 0 and not args.no_carry) else 0
        h = optim.native_hparams(hp, st, lr=0.01, grad_scale=1.0 / 32768, flags=flags)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        nat.check(lib.lars_step(plan.handle, _ptr(params.param_shard), _ptr(params.grad_shard_of_full),
                                _ptr(params.momentum), nat.ctypes.byref(h), _ptr(eng.d_iter),
                                _ptr(eng.d_sumsq), _ptr(eng.d_lambda), _ptr(eng.d_info), _ptr(ws),
                                _stream()))
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    print("event-timed step (last 3):", [round(a.elapsed_time(b) * 1e3, 2) for a, b in ev[-3:]], "us")
    lib.lars_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    nw = plan.info.grid * 8
    buf = np.zeros(nw * 8, dtype=np.uint64)
    nat.check(lib.lars_debug_trace(buf.ctypes.data, buf.size))
    raw = buf.reshape(nw, 8)
    smid = raw[:, 7].astype(np.int64)
    t = raw[:, :5].astype(np.int64)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3  # us
    def q(x):
        return f"min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f}"
    print(f"grid {plan.info.grid} warps {nw} params {params.shard_numel} pieces {plan.info.npieces}")
    print(f"kernel span (first warp start -> last warp end): {t[:, 4].max():.2f} us")
    if os.environ.get("TRACE_DUMP"):
        np.save(os.environ["TRACE_DUMP"], raw)
    print("start        ", q(t[:, 0]))
    print("phase A      ", q(t[:, 1] - t[:, 0]))
    print("A end        ", q(t[:, 1]))
    print("barrier exit ", q(t[:, 2]))
    print("coef ready   ", q(t[:, 3]))
    print("barrier wait ", q(t[:, 2] - t[:, 1]), " (per warp: exit - own A end)")
    print("lambda       ", q(t[:, 3] - t[:, 2]), " (per warp: coef ready - exit)")
    t56 = (raw[:, 5:7].astype(np.int64) - t0) / 1e3
    if (raw[:, 5] > 0).all():
        print("  staged     ", q(t56[:, 0] - t[:, 2]), " (per warp: partials staged - exit)")
        print("  computed   ", q(t56[:, 1] - t56[:, 0]), " (per warp: lambda loop)")
        print("  sync       ", q(t[:, 3] - t56[:, 1]))
    print("phase B      ", q(t[:, 4] - t[:, 3]))
    print("B end        ", q(t[:, 4]))
    pb = t[:, 4] - t[:, 3]
    cta = np.arange(nw) // 8
    wic = np.arange(nw) % 8
    print("phase B by warp-in-CTA:", [round(float(pb[wic == k].mean()), 1) for k in range(8)])
    print("phase B by CTA parity:", [round(float(pb[cta % 2 == k].mean()), 1) for k in range(2)])
    print("phase B by CTA half:", [round(float(pb[(cta >= plan.info.grid // 2) == k].mean()), 1) for k in range(2)])
    sm_mean = {}
    for sm in np.unique(smid):
        sm_mean[int(sm)] = float(pb[smid == sm].mean())
    v = np.array(list(sm_mean.values()))
    print(f"phase B per-SM mean: min {v.min():.1f} med {np.median(v):.1f} max {v.max():.1f} over {len(v)} SMs")
    order = sorted(sm_mean, key=sm_mean.get)
    print("fastest SMs", order[:12], "slowest SMs", order[-12:])
    pa = t[:, 1] - t[:, 0]
    va = np.array([pa[smid == sm].mean() for sm in order])
    print("phase A per-SM (same order):", np.round(va[:6], 1), np.round(va[-6:], 1))
    # %globaltimer may be offset between the two dies: end times per SM half
    for name, sel in (("SM < 74", smid < 74), ("SM >= 74", smid >= 74)):
        if sel.any():
            print(f"{name}: start med {np.median(t[sel, 0]):.2f}  A end max {t[sel, 1].max():.2f}  "
                  f"barrier exit min {t[sel, 2].min():.2f}  B end min {t[sel, 4].min():.2f} "
                  f"max {t[sel, 4].max():.2f}")
    # per-CTA view (how the last phase-A straggler pattern was found): the
    # slowest warp of each CTA, averaged per tenth of the grid
    cta_pa = (t[:, 1] - t[:, 0]).reshape(-1, 8).max(axis=1)
    tenth = max(1, len(cta_pa) // 10)
    print("phase A per CTA, by tenth of the grid:",
          [round(float(cta_pa[i * tenth:(i + 1) * tenth].mean()), 2) for i in range(10)],
          "slowest CTAs:", [int(c) for c in np.argsort(cta_pa)[-6:]])
    # within-SM spread
    spread = [float(pb[smid == sm].max() - pb[smid == sm].min()) for sm in order]
    print("within-SM phase-B spread: med", round(float(np.median(spread)), 1), "max", round(max(spread), 1))


if __name__ == "__main__":
    main()
