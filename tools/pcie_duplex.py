"""PCIe copy bandwidth of this box: host-to-device alone, device-to-host
alone, and both at once on two streams (pinned host buffers, 256 MiB each).

    python tools/pcie_duplex.py
"""
import torch

n = 64 << 20  # float32 elements: 256 MiB
dev = torch.device("cuda:0")
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device=dev)
d_out = torch.ones(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


gb = 4 * n / 1e9
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D alone {gb / t1:6.1f} GB/s | D2H alone {gb / t2:6.1f} GB/s | "
      f"both at once {2 * gb / t3:6.1f} GB/s aggregate ({t3 * 1e3:.2f} ms vs {(t1 + t2) * 1e3:.2f} ms serial)")

# the same with numpy memory registered in place (cudaHostRegister, 4 KiB
# pages), as the host ParamSet path uses for the caller's arrays
import ctypes  # noqa: E402
import os  # noqa: E402
import sys  # noqa: E402

import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_05011_b200 import _native as nat  # noqa: E402

lib = nat.load()
a_in = np.ones(n, dtype=np.float32)
a_out = np.empty(n, dtype=np.float32)
for arr in (a_in, a_out):
    nat.check(lib.lars_host_register(ctypes.c_void_p(arr.ctypes.data), arr.nbytes))
h_in = torch.from_numpy(a_in)
h_out = torch.from_numpy(a_out)
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"registered numpy: H2D alone {gb / t1:6.1f} GB/s | D2H alone {gb / t2:6.1f} GB/s | "
      f"both at once {2 * gb / t3:6.1f} GB/s aggregate")
