"""Per-warp timeline of the streamed sharded step (torchrun, trace build).

    python -m paper_1709_05011_b200.build --trace
    torchrun --nproc-per-node 2 tools/trace_stream.py [--workload resnet50]

Per rank: when the A-workers (reduce-scatter) finish, when the B-workers
(update + all-gather) get their first segment and finish, how long B-workers
waited for segments in total, and the kernel span -- i.e. how much the two
NVLink directions overlapped.
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
ap.add_argument("--awarps", type=int, default=4, help="A-worker warps per CTA of the build")
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
params = FlatParamSet(layouts.get(args.workload), dev, world_size=world, rank=rank, symmetric=True)
g = torch.Generator(device=dev)
g.manual_seed(1 + rank)
for grp in params:
    grp.param.uniform_(-0.05, 0.05, generator=g)
    grp.grad.normal_(0, 1.0, generator=g)
hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5, lars_enabled=True)
st = optim.ScheduleState(3515, 39)
dp = DataParallelLars(params, backend="p2p-stream")
flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
for _ in range(args.steps):
    flush.zero_()
    dist.barrier(device_ids=[rank])
    dp.step(hp, st, grad_scale=1.0 / 32768)
torch.cuda.synchronize()
lib = nat.load()
lib.lars_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
plan, _ = params.engine().plan(frozenset(hp.lars_skip_categories))
nw = plan.info.grid * 8
buf = np.zeros(nw * 8, dtype=np.uint64)
nat.check(lib.lars_debug_trace(buf.ctypes.data, buf.size))
raw = buf.reshape(nw, 8).astype(np.int64)
t0 = raw[:, 0].min()
ts = lambda k: (raw[:, k] - t0) / 1e3  # noqa: E731
is_a = (np.arange(nw) % 8) < args.awarps
a_end = ts(1)[is_a]
b_first = ts(3)
b_end = ts(4)
end = ts(5)
wait = raw[:, 6] / 1e3
stats = [ts(2).max(), np.median(a_end), a_end.max(), np.median(b_first[~is_a]), np.median(b_end),
         b_end.max(), end.max(), np.median(wait[~is_a]), np.median(wait[is_a])]
mine = torch.tensor(stats, dtype=torch.float64, device=dev)
allr = [torch.zeros_like(mine) for _ in range(world)]
dist.all_gather(allr, mine)
if rank == 0:
    print(f"{args.workload} world {world}: shard {params.shard_numel} params, grid {plan.info.grid}, "
          f"A-warps {args.awarps}/8")
    for r, v in enumerate(allr):
        v = v.tolist()
        print(f"rank {r}: start barrier {v[0]:6.1f} | A end med {v[1]:6.1f} max {v[2]:6.1f} | "
              f"B first chunk med {v[3]:6.1f} | B end med {v[4]:6.1f} max {v[5]:6.1f} | "
              f"kernel end {v[6]:6.1f} | B wait med (B-warps) {v[7]:6.1f} (A-warps) {v[8]:6.1f} us")
dist.barrier(device_ids=[rank])
dist.destroy_process_group()
