"""Kernel-only strong scaling on ONE GPU: time the fused lars_step kernel on
every rank's shard plan of a world of P ranks (P = 1, 2, 4, 8), so
E_k(P) = T(full set) / (P * max_r T(shard r)) (definition 1)
is measurable without P GPUs.  Inputs as bench.py (L2 flushed before each
launch, carry on after the first launch, CUDA events on the launching stream).

    python tools/shard_time.py [--workloads resnet50,alexnet_bn,sweep:1e6:50]
                               [--worlds 1,2,4,8] [--reps 30] [--lib NAME]

Prints one JSON line per (workload, P) and a summary line.
"""
import argparse
import json
import os
import statistics
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def time_shard(layout, world, rank, reps, flush, dev, grid=0):
    import torch
    from paper_1709_05011_b200 import _native as nat
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.flat import FlatParamSet, _ptr
    params = FlatParamSet(layout, dev, world_size=world, rank=rank)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    for grp in params:
        if grp.category == "norm-scale":
            grp.param.fill_(1.0)
        elif grp.category == "weight":
            grp.param.uniform_(-0.05, 0.05, generator=g)
        grp.grad.normal_(0.0, 32.768, generator=g)
    hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5,
                           lars_enabled=True)
    st = optim.ScheduleState(3515, 39)
    eng = params.engine()
    if grid:
        from paper_1709_05011_b200.flat import _Plan
        plan = _Plan(params.segments(), len(params), frozenset(hp.lars_skip_categories), grid=grid)
        ws = torch.empty(int(plan.info.workspace_bytes), dtype=torch.uint8, device=dev)
        nat.check(nat.load().lars_workspace_init(plan.handle, _ptr(ws), torch.cuda.current_stream().cuda_stream))
    else:
        plan, ws = eng.plan(frozenset(hp.lars_skip_categories))
    lib = nat.load()
    stream = torch.cuda.current_stream()
    w, gr, m = params.param_shard, params.grad_shard_of_full, params.momentum
    ts = []
    for i in range(reps + 3):
        flags = nat.LARS_STEP_USE_WCARRY if i > 0 else 0
        h = optim.native_hparams(hp, st, lr=0.01, grad_scale=1.0 / 32768, flags=flags)
        flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nat.check(lib.lars_step(plan.handle, _ptr(w), _ptr(gr), _ptr(m), nat.ctypes.byref(h),
                                _ptr(eng.d_iter), _ptr(eng.d_sumsq), _ptr(eng.d_lambda),
                                _ptr(eng.d_info), _ptr(ws), stream.cuda_stream))
        b.record(stream)
        if i >= 3:
            ts.append((a, b))
    torch.cuda.synchronize()
    us = statistics.median([a.elapsed_time(b) for a, b in ts]) * 1e3
    return us, params.shard_numel, int(plan.info.grid)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="resnet50,alexnet_bn,sweep:1e6:50,sweep:16e6:100")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--grid", type=int, default=0, help="CTAs per launch (0: the plan default)")
    args = ap.parse_args()
    import torch
    from paper_1709_05011_b200 import layouts
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    fbuf = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    cbuf = torch.ones(1 << 26, dtype=torch.float32, device=dev)

    def flush():
        fbuf.zero_()
        cbuf.sum()

    peak = 6536.0
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    summary = {}
    for wl in args.workloads.split(","):
        layout = layouts.get(wl)
        t1 = None
        for P in [int(x) for x in args.worlds.split(",")]:
            per = [time_shard(layout, P, r, args.reps, flush, dev, args.grid) for r in range(P)]
            tmax = max(p[0] for p in per)
            n_shard = per[0][1]
            if P == 1:
                t1 = tmax
            line = {"workload": wl, "P": P, "shard_params": n_shard,
                    "t_us": [round(p[0], 2) for p in per], "t_max_us": round(tmax, 2),
                    "frac_hbm_max": round(20 * n_shard / (tmax * 1e-6) / 1e9 / peak, 4),
                    "grid": per[0][2]}
            if t1 is not None:
                line["E_k"] = round(t1 / (P * tmax), 4)
            summary[f"{wl}:P{P}"] = line.get("E_k")
            print(json.dumps(line), flush=True)
            torch.cuda.empty_cache()
    print(json.dumps({"summary_E_k": summary}), flush=True)


if __name__ == "__main__":
    main()
