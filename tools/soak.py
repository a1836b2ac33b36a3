"""Race soak: the same long run twice must give bitwise identical weights.

    python tools/soak.py [--steps 1000] [--workload resnet50]                  # 1 GPU, fused step
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/soak.py --steps 500   # p2p step

Every step draws a fresh seeded gradient on the device; the kernel is
deterministic by construction (fixed reduction orders), so any difference
between the two runs -- or between ranks -- means a visibility race (a
barrier or fence that let stale data through).  Prints one JSON line.
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1709_05011_b200 import layouts, optim  # noqa: E402
from paper_1709_05011_b200.cluster import DataParallelLars, check_synchronized  # noqa: E402
from paper_1709_05011_b200.flat import FlatParamSet  # noqa: E402


def run(layout, steps, world, rank, dev, backend="auto"):
    params = FlatParamSet(layout, dev, world_size=world, rank=rank, symmetric=world > 1)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for grp in params:
        grp.param.uniform_(-0.05, 0.05, generator=g)
    params.invalidate_norm_cache()
    hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5,
                           lars_enabled=True)
    st = optim.ScheduleState(10 ** 6, 39)
    dp = DataParallelLars(params, backend=backend if world > 1 else "auto")
    lam_digest = hashlib.sha256()
    for t in range(steps):
        g.manual_seed(1000 + 7919 * t + rank)
        params.flat_grad.normal_(0.0, 32.0, generator=g)
        lams = dp.step(hp, st, grad_scale=1.0 / 32768)
        if t % 50 == 49:
            lam_digest.update(repr(dict(lams)).encode())
    torch.cuda.synchronize()
    if world > 1:
        check_synchronized(params)
    w = hashlib.sha256(params.flat_param.cpu().numpy().tobytes()).hexdigest()
    m = hashlib.sha256(params.momentum.cpu().numpy().tobytes()).hexdigest()
    return w, m, lam_digest.hexdigest(), dp.backend


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--backend", default="auto")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    layout = layouts.get(args.workload)
    a = run(layout, args.steps, world, rank, dev, args.backend)
    b = run(layout, args.steps, world, rank, dev, args.backend)
    ok = a == b
    res = torch.tensor([1 if ok else 0], device=dev)
    if world > 1:
        dist.all_reduce(res, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"soak": args.workload, "world": world, "steps": args.steps,
                          "backend": a[3], "runs_identical_on_all_ranks": bool(res.item()),
                          "w_sha256": a[0][:16]}), flush=True)
    if world > 1:
        dist.barrier()
        os._exit(0 if res.item() else 1)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
