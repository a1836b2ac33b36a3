"""Per-warp phase timeline of the peer-memory fused sharded step (torchrun, trace build).

    python -m paper_1709_05011_b200.build --trace
    torchrun --nproc-per-node 2 tools/trace_nvls.py [--workload resnet50]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LARS_B200_LIB", "liblars_b200_trace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1709_05011_b200 import _native as nat, layouts, optim  # noqa: E402
from paper_1709_05011_b200.cluster import DataParallelLars  # noqa: E402
from paper_1709_05011_b200.flat import FlatParamSet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="resnet50")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--overlap", action="store_true",
                help="ResNet-50 module + BackwardOverlap: the step reduces from local receive slots")
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
if args.overlap:
    from paper_1709_05011_b200.train import build_model
    model = build_model("resnet50").to(dev)
    params = FlatParamSet.from_module(model, dev, world_size=world, rank=rank, symmetric=True)
else:
    layout = layouts.get(args.workload)
    params = FlatParamSet(layout, dev, world_size=world, rank=rank, symmetric=True)
g = torch.Generator(device=dev)
g.manual_seed(1 + rank)
for grp in params:
    grp.param.uniform_(-0.05, 0.05, generator=g)
    grp.grad.normal_(0, 1.0, generator=g)
hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5, lars_enabled=True)
st = optim.ScheduleState(3515, 39)
dp = DataParallelLars(params, backend="p2p")
assert dp.backend == "p2p"
ov = dp.overlap_backward(model) if args.overlap else None
flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
for _ in range(args.steps):
    flush.zero_()
    dist.barrier(device_ids=[rank])
    if ov is not None:
        # no backward here: push every bucket before the step (as the hooks
        # would during backward), then the step reduces from the local slots
        ov.arm()
        ov.push_all()
        torch.cuda.synchronize()
        dist.barrier(device_ids=[rank])
    dp.step(hp, st, grad_scale=1.0 / 32768)
torch.cuda.synchronize()
lib = nat.load()
if not hasattr(lib, "lars_debug_trace"):  # a non-trace build: just the steps (e.g. under ncu)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0)
lib.lars_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
plan, _ = params.engine().plan(frozenset(hp.lars_skip_categories))
nw = plan.info.grid * 8
buf = np.zeros(nw * 8, dtype=np.uint64)
nat.check(lib.lars_debug_trace(buf.ctypes.data, buf.size))
raw = buf.reshape(nw, 8).astype(np.int64)
if os.environ.get("TRACE_DUMP"):
    np.save(f"{os.environ['TRACE_DUMP']}_r{rank}.npy", raw)
t = raw[:, :7]
t = (t - t[:, 0].min()) / 1e3
# every rank: its own phase-A end spread and exchange timing (relative to its start)
mine = torch.tensor([t[:, 1].max(), t[:, 1].min(), t[0, 2], t[0, 5], t[0, 6], t[0, 3], t[:, 4].max(),
                     float(raw[:, 0].min() % 10**9) / 1e3], dtype=torch.float64, device=dev)
allr = [torch.zeros_like(mine) for _ in range(world)]
dist.all_gather(allr, mine)
if rank == 0:
    for r, v in enumerate(allr):
        v = v.tolist()
        print(f"rank {r}: A end min {v[1]:7.2f} max {v[0]:7.2f} | cta0 barrier1 {v[2]:7.2f} sums stored {v[3]:7.2f}"
              f" rank-barrier exit {v[4]:7.2f} coef {v[5]:7.2f} | B end max {v[6]:7.2f} | start(abs us mod 1s) {v[7]:.2f}")
if rank == 0:
    q = lambda x: f"min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f}"  # noqa: E731
    print(f"rank {rank} grid {plan.info.grid} shard {params.shard_numel}")
    for k, name in [(0, "start"), (1, "A end"), (2, "barrier1 exit"), (3, "coef ready"), (4, "B end")]:
        print(f"{name:14s}", q(t[:, k]))
    print(f"{'start barrier':14s}", q(t[1:, 5] - t[1:, 0]), " (per warp: exit - own start)")
    # CTA 0 / warp 0: norm exchange (local sums stored to the peers, rank barrier)
    print(f"cta0 A end {t[0, 1]:.2f}  barrier1 exit {t[0, 2]:.2f}  sums stored {t[0, 5]:.2f}  "
          f"rank barrier exit {t[0, 6]:.2f}  coef ready {t[0, 3]:.2f}")
dist.barrier()
os._exit(0)
