"""NVLink / NVLS throughput on this box (torchrun, N ranks): multimem.ld_reduce,
multimem.st, P2P read and write of a 256 MB buffer.  Prints GB/s per rank."""
import ctypes
import os
import subprocess
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "_nvls_bw.so")
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
if rank == 0 and not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", os.path.join(HERE, "nvls_bw.cu"), "-o", so])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
dist.barrier()
lib = ctypes.CDLL(so)
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
n = 64 << 20  # floats = 256 MB
t = symm_mem.empty(n, dtype=torch.float32, device=dev)
t.fill_(1.0)
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
mc = int(h.multicast_ptr) + (t.data_ptr() - int(h.buffer_ptrs[h.rank]))
peer = int(h.buffer_ptrs[(rank + 1) % world])
out = torch.zeros(1, device=dev)
st = torch.cuda.current_stream()
res = {}
def grids(which):
    return (148, 296, 444) if which == 4 else (148 * 4, 148 * 8)


for name, which, ptr in [("ld_reduce", 0, mc), ("mc_store", 1, mc), ("p2p_read", 2, peer),
                         ("p2p_write", 3, peer), ("bulk_read", 4, peer)]:
    for grid in grids(which):
        times = []
        for it in range(6):
            dist.barrier(device_ids=[rank])
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            assert lib.run(which, ctypes.c_void_p(ptr), n // 4, ctypes.c_void_p(out.data_ptr()), grid, 256, ctypes.c_void_p(st.cuda_stream)) == 0
            b.record(st)
            b.synchronize()
            if it >= 2:
                times.append(a.elapsed_time(b))
        ms = min(times)
        res[(name, grid)] = n * 4 / (ms * 1e-3) / 1e9
# copy engines (cudaMemcpyAsync D2D through the peer mapping)
peer_t = h.get_buffer((rank + 1) % world, (n,), torch.float32,
                      (t.data_ptr() - int(h.buffer_ptrs[h.rank])) // 4)
local = torch.empty(n, dtype=torch.float32, device=dev)
for name, fn in [("ce_read", lambda: local.copy_(peer_t, non_blocking=True)),
                 ("ce_write", lambda: peer_t.copy_(local, non_blocking=True))]:
    times = []
    for it in range(6):
        dist.barrier(device_ids=[rank])
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        if it >= 2:
            times.append(a.elapsed_time(b))
    res[(name, 0)] = n * 4 / (min(times) * 1e-3) / 1e9
# SM peer reads and a copy-engine peer read running concurrently (two streams),
# each on half of the buffer: does the link carry more than either alone?
side = torch.cuda.Stream()
half = n // 2
for grid in (148 * 2, 148 * 4):
    times = []
    for it in range(6):
        dist.barrier(device_ids=[rank])
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        side.wait_stream(st)
        with torch.cuda.stream(side):
            local[half:].copy_(peer_t[half:], non_blocking=True)
        assert lib.run(2, ctypes.c_void_p(peer), half // 4, ctypes.c_void_p(out.data_ptr()), grid, 256,
                       ctypes.c_void_p(st.cuda_stream)) == 0
        st.wait_stream(side)
        b.record(st)
        b.synchronize()
        if it >= 2:
            times.append(a.elapsed_time(b))
    res[("sm+ce_read", grid)] = n * 4 / (min(times) * 1e-3) / 1e9
dist.barrier(device_ids=[rank])
if rank == 0:
    for k, v in res.items():
        print(f"world {world} {k[0]:10s} grid {k[1]:5d}: {v:8.1f} GB/s (bytes of the buffer / time)")
sys.stdout.flush()
os._exit(0)
