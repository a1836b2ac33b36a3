"""Exposed optimizer time of the ResNet-50 data-parallel step, with and
without the backward-overlapped gradient push (overlap.py).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/overlap_time.py

Per step (one micro-batch of 256 per rank, bf16 autocast): events right
after `loss.backward()` is queued and after `dp.step()`; their difference is
the time from the end of backward on the GPU to the end of the step, i.e.
what the optimizer adds to the step (max over ranks, median over steps).
Also prints the whole step time.  Prints one JSON line on rank 0.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1709_05011_b200 import optim  # noqa: E402
from paper_1709_05011_b200.train import Trainer, build_model  # noqa: E402


BUCKET = int(float(os.environ.get("OVERLAP_BUCKET_MB", 16)) * (1 << 20))


def run(overlap, steps, micro):
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.manual_seed(0)
    gb = micro * world
    hp = optim.HyperParams(base_lr=optim.linear_scaled_lr(0.2, 256, gb), epochs=90, batch_size=gb,
                           warmup_epochs=5, lars_enabled=True)
    st = optim.ScheduleState(10 ** 6, 10 ** 4)
    tr = Trainer(build_model("resnet50"), hp, st, gb, micro, dev, "p2p")
    if overlap:
        tr.overlap = tr.dp.overlap_backward(tr.model, bucket_bytes=BUCKET)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(micro, 3, 224, 224, device=dev, generator=g).to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (micro,), device=dev, generator=g)
    exposed, whole = [], []
    for i in range(steps + 3):
        tr.params.zero_grads()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = tr.model(x)
        loss = tr.loss(out.float(), y)
        if tr.overlap is not None:
            tr.overlap.arm()
        loss.backward()
        e1.record()
        tr.dp.step(hp, st, grad_scale=1.0 / gb)
        e2.record()
        e2.synchronize()
        if i >= 3:
            exposed.append(e1.elapsed_time(e2) * 1e3)
            whole.append(e0.elapsed_time(e2) * 1e3)
    t = torch.tensor([statistics.median(exposed), statistics.median(whole)], device=dev)
    lo = t.clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    if tr.overlap is not None:
        tr.overlap.remove()
    # max over ranks includes waiting for the rank whose backward ends last;
    # min over ranks (that last rank) is the step's own exposed time
    return float(t[0]), float(lo[0]), float(t[1])


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.backends.cudnn.benchmark = True
    steps = int(os.environ.get("OVERLAP_STEPS", 10))
    res = {}
    for mode in (False, True, False, True):
        ex, ex_lo, wh = run(mode, steps, 256)
        res.setdefault("overlap" if mode else "plain", []).append(
            {"exposed_max_us": round(ex, 1), "exposed_min_us": round(ex_lo, 1),
             "step_us": round(wh, 1)})
    if dist.get_rank() == 0:
        print(json.dumps({"world": dist.get_world_size(), "micro_batch": 256,
                          "bucket_mb": BUCKET >> 20, "runs": res}), flush=True)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
