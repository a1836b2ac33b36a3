"""Flat, layer-segmented parameter storage: the boundary type of the step.

`FlatParamSet` is the device-resident counterpart of the reference
`nn.ParamSet` (pkg/src/batchlab/nn.py:72-114): ordered, uniquely named
parameter groups, each with `param`, `grad`, `momentum_buf` and `category`
(nn.py:63-69), and the same methods (`names`, `zero_grads`, `set_grads`,
`copy`, `checksum`).  The difference is the storage: every group is a view
into three flat fp32 buffers (weights, gradients, momentum), each group
starting on a 128-byte boundary with zero padding after it, so one kernel
launch can sweep the whole set with 16-byte vector loads.

For a data-parallel world of P ranks the flat length is padded to a multiple
of 32*P and split into P equal contiguous shards (what NCCL reduce-scatter /
all-gather need).  Rank r owns elements [r*C, (r+1)*C): its momentum is
stored only for that shard (ZeRO-1 style; the reference keeps a full
momentum replica per worker, cluster.py:151-153), and its step plan covers
the layer pieces inside the shard.
"""

import hashlib
import struct
import weakref

import numpy as np
import torch

from . import _native as nat
from .errors import ConfigError, DivergenceError
from .layouts import BIAS, NORM_SCALE, NORM_SHIFT, WEIGHT, numel

ALIGN = 32  # elements: 128 bytes


def _round_up(x, m):
    return ((x + m - 1) // m) * m


class ParamGroup:
    """One named group; mirrors nn.ParamGroup (nn.py:63-69).

    `param` / `grad` are views into the flat buffers; `momentum_buf` is a
    view into the momentum buffer when this rank holds the whole set, else
    None (the momentum of a sharded set lives in `FlatParamSet.momentum`).
    """

    __slots__ = ("name", "param", "grad", "momentum_buf", "category", "index", "offset",
                 "numel", "shape")

    def __init__(self, name, param, grad, momentum_buf, category, index, offset, n, shape):
        self.name = name
        self.param = param
        self.grad = grad
        self.momentum_buf = momentum_buf
        self.category = category
        self.index = index
        self.offset = offset
        self.numel = n
        self.shape = shape

    def __repr__(self):
        return f"ParamGroup({self.name!r}, shape={tuple(self.shape)}, category={self.category!r})"


class FlatParamSet:
    """Ordered parameter groups over flat fp32 device buffers."""

    def __init__(self, layout, device=None, *, world_size=1, rank=0, symmetric=False):
        layout = [(str(n), tuple(int(d) for d in s), str(c)) for n, s, c in layout]
        names = [n for n, _, _ in layout]
        if len(set(names)) != len(names):  # nn.py:77-79
            raise ConfigError(f"duplicate parameter group names: {names}")
        if not layout:
            raise ConfigError("empty parameter set")
        if world_size < 1 or not 0 <= rank < world_size:
            raise ConfigError(f"bad rank {rank} for world size {world_size}")
        self.device = torch.device(device if device is not None else "cuda")
        self.layout = layout
        self.world_size = world_size
        self.rank = rank
        offsets = []
        off = 0
        for _, shape, _ in layout:
            off = _round_up(off, ALIGN)
            offsets.append(off)
            off += numel(shape)
        self.numel = sum(numel(s) for _, s, _ in layout)
        self.padded_numel = _round_up(max(off, 1), ALIGN * world_size)
        self.shard_numel = self.padded_numel // world_size
        self.shard_lo = rank * self.shard_numel
        self.shard_hi = self.shard_lo + self.shard_numel
        dev = self.device
        self.symmetric = bool(symmetric)
        if self.symmetric:
            # weights and gradients in symmetric (multicast-capable) memory for
            # the peer-memory fused sharded step (cluster.DataParallelLars(backend="p2p"))
            import torch.distributed._symmetric_memory as symm_mem
            self.flat_param = symm_mem.empty(self.padded_numel, dtype=torch.float32, device=dev)
            self.flat_grad = symm_mem.empty(self.padded_numel, dtype=torch.float32, device=dev)
            self.flat_param.zero_()
            self.flat_grad.zero_()
        else:
            self.flat_param = torch.zeros(self.padded_numel, dtype=torch.float32, device=dev)
            self.flat_grad = torch.zeros(self.padded_numel, dtype=torch.float32, device=dev)
        self.momentum = torch.zeros(self.shard_numel, dtype=torch.float32, device=dev)
        self.groups = []
        for i, ((name, shape, cat), o) in enumerate(zip(layout, offsets)):
            n = numel(shape)
            p = self.flat_param[o:o + n].view(shape)
            g = self.flat_grad[o:o + n].view(shape)
            m = self.momentum[o:o + n].view(shape) if world_size == 1 else None
            self.groups.append(ParamGroup(name, p, g, m, cat, i, o, n, shape))
        self._by_name = {g.name: g for g in self.groups}
        self._engine = None
        # module parameters bound to the flat buffers by from_module: writes
        # through them (p.mul_, load_state_dict) bump their own version
        # counters, not flat_param's, so the norm carry checks them too
        self._bound = ()
        self._dp = None  # cluster.global_step's DataParallelLars

    # ---- nn.ParamSet surface (nn.py:81-114) --------------------------------
    def __iter__(self):
        return iter(self.groups)

    def __len__(self):
        return len(self.groups)

    def __getitem__(self, name):
        return self._by_name[name]

    def names(self):
        return [g.name for g in self.groups]

    def zero_grads(self):
        self.flat_grad.zero_()

    def set_grads(self, grads):
        """Copy gradients in: a name -> array mapping (nn.py:98-101) or one flat
        tensor of `padded_numel` elements (e.g. a pinned host buffer)."""
        if isinstance(grads, torch.Tensor) and grads.dim() == 1 and grads.numel() == self.padded_numel:
            self.flat_grad.copy_(grads, non_blocking=True)
            return
        for g in self.groups:
            src = grads[g.name]
            if not isinstance(src, torch.Tensor):
                src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32))
            g.grad.copy_(src.reshape(g.shape), non_blocking=True)

    def shard_slices(self, name):
        """(slice into `momentum`, slice into the group's flattened values)
        of the part of group `name` this rank owns, or None."""
        g = self._by_name[name]
        a = max(g.offset, self.shard_lo)
        b = min(g.offset + g.numel, self.shard_hi)
        if b <= a:
            return None
        return slice(a - self.shard_lo, b - self.shard_lo), slice(a - g.offset, b - g.offset)

    def set_momentum(self, name, values):
        """Load a group's momentum (this rank's part of it when sharded)."""
        sl = self.shard_slices(name)
        if sl is not None:
            self.momentum[sl[0]].copy_(_as_tensor(values).reshape(-1)[sl[1]])
        self.invalidate_norm_cache()

    def get_momentum(self, name):
        """This rank's part of a group's momentum, flattened (None if none)."""
        sl = self.shard_slices(name)
        return None if sl is None else self.momentum[sl[0]]

    def copy(self):
        twin = FlatParamSet(self.layout, self.device, world_size=self.world_size, rank=self.rank,
                            symmetric=self.symmetric)
        twin.flat_param.copy_(self.flat_param)
        twin.flat_grad.copy_(self.flat_grad)
        twin.momentum.copy_(self.momentum)
        return twin

    def checksum(self):
        """SHA-256 over names and parameter bytes, like nn.ParamSet.checksum
        (nn.py:109-114); the bytes are the fp32 device values."""
        host = self.flat_param.detach().cpu().numpy()
        h = hashlib.sha256()
        for g in self.groups:
            h.update(g.name.encode())
            h.update(np.ascontiguousarray(host[g.offset:g.offset + g.numel]).tobytes())
        return h.hexdigest()

    def fingerprint(self):
        """Cheap on-device replica fingerprint (two int64 sums of the fp32 bit
        patterns) used by the cross-rank synchronisation check."""
        bits = self.flat_param.view(torch.int32).to(torch.int64)
        pos = torch.arange(1, bits.numel() + 1, device=bits.device, dtype=torch.int64)
        return torch.stack([bits.sum(), (bits * pos).sum()])

    # ---- construction helpers ---------------------------------------------
    @classmethod
    def from_groups(cls, groups, device=None, **kw):
        """From reference-style groups (objects with name/param/grad/
        momentum_buf/category, e.g. a reference nn.ParamSet): values copied
        in as fp32."""
        groups = list(groups)
        layout = [(g.name, tuple(np.shape(g.param)), g.category) for g in groups]
        fps = cls(layout, device, **kw)
        fps.load_groups(groups)
        return fps

    def load_groups(self, groups, momentum=True):
        for src in groups:
            dst = self._by_name[src.name]
            dst.param.copy_(_as_tensor(src.param).reshape(dst.shape))
            dst.grad.copy_(_as_tensor(src.grad).reshape(dst.shape))
            if momentum and src.momentum_buf is not None:
                if dst.momentum_buf is None:
                    raise ConfigError("momentum of a sharded set lives in .momentum")
                dst.momentum_buf.copy_(_as_tensor(src.momentum_buf).reshape(dst.shape))
        self.invalidate_norm_cache()

    def store_groups(self, groups):
        """Write param and momentum back into reference-style numpy groups."""
        w = self.flat_param.detach().cpu().numpy()
        m = self.momentum.detach().cpu().numpy()
        for dst in groups:
            src = self._by_name[dst.name]
            np.copyto(dst.param, w[src.offset:src.offset + src.numel].reshape(np.shape(dst.param)))
            if self.world_size == 1:
                np.copyto(dst.momentum_buf,
                          m[src.offset:src.offset + src.numel].reshape(np.shape(dst.param)))

    @classmethod
    def from_module(cls, module, device=None, **kw):
        """Move a torch module's parameters into flat storage: each
        `p.data` / `p.grad` becomes a view of the flat buffers, so backward
        accumulates straight into the flat gradient (call `zero_grads()`, not
        `module.zero_grad(set_to_none=True)`)."""
        layout, params = [], []
        for full, mod, pname, p in _module_params(module):
            layout.append((full, tuple(p.shape), _category(mod, pname)))
            params.append(p)
        fps = cls(layout, device or (params[0].device if params else None), **kw)
        with torch.no_grad():
            for grp, p in zip(fps.groups, params):
                grp.param.copy_(p.detach())
                p.data = grp.param
                p.grad = grp.grad
        fps._bound = tuple(params)
        fps.invalidate_norm_cache()
        return fps

    # ---- plan / step plumbing ---------------------------------------------
    def segments(self):
        """Segment table of this rank's shard (offsets relative to shard_lo),
        one per group, zero-length where the group lies outside the shard."""
        segs = []
        for g in self.groups:
            lo = g.offset
            hi = g.offset + _round_up(g.numel, 4)
            a, b = max(lo, self.shard_lo), min(hi, self.shard_hi)
            segs.append((a - self.shard_lo if b > a else 0, max(0, b - a), g.index, g.category))
        return segs

    def shared_flags(self):
        """Per segment of segments(): does the group also have elements in
        another rank's shard (its norms need the other ranks' sums)?"""
        out = []
        for g in self.groups:
            lo, hi = g.offset, g.offset + _round_up(g.numel, 4)
            out.append(self.world_size > 1 and (lo < self.shard_lo or hi > self.shard_hi)
                       and min(hi, self.shard_hi) > max(lo, self.shard_lo))
        return out

    def invalidate_norm_cache(self):
        """Forget the carried ||w||^2 of the last step.  Writes through
        `flat_param`, its views or the module parameters bound by
        `from_module` are detected (tensor version counters); call this after
        any other write to the weights (raw pointers, another library)."""
        if self._engine is not None:
            self._engine.invalidate()

    def weights_version(self):
        """Version stamp of every tensor through which the weights can be
        written: the flat buffer (its views share its counter) and the bound
        module parameters."""
        v = self.flat_param._version
        for p in self._bound:
            v += p._version
        return v

    def engine(self):
        if self._engine is None:
            self._engine = LarsEngine(self)
        return self._engine

    # local shard views (what the step kernels touch)
    @property
    def param_shard(self):
        return self.flat_param[self.shard_lo:self.shard_hi]

    @property
    def grad_shard_of_full(self):
        return self.flat_grad[self.shard_lo:self.shard_hi]


def _as_tensor(x):
    if isinstance(x, torch.Tensor):
        return x.detach().to(torch.float32)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))


def _category(mod, pname):
    norm_types = (torch.nn.modules.batchnorm._NormBase, torch.nn.LayerNorm, torch.nn.GroupNorm)
    if isinstance(mod, norm_types):
        return NORM_SCALE if pname == "weight" else NORM_SHIFT
    return BIAS if pname == "bias" else WEIGHT


# ---------------------------------------------------------------------------
# LarsEngine: the plan, workspace and device-side scalars of one shard
# ---------------------------------------------------------------------------

def _module_params(module):
    for mod_name, mod in module.named_modules():
        for pname, p in mod.named_parameters(recurse=False):
            yield (f"{mod_name}.{pname}" if mod_name else pname), mod, pname, p


def module_parameters(module):
    """The module's parameters in FlatParamSet.from_module group order."""
    return [p for _, _, _, p in _module_params(module)]


_DEFERRED_PLANS = []


def _capturing():
    return torch.cuda.is_available() and torch.cuda.is_initialized() and \
        torch.cuda.is_current_stream_capturing()


def _destroy_plan(lib, handle):
    """Plan destructor.  lars_plan_destroy frees device memory, which is
    illegal while a CUDA graph is being captured (a garbage-collected plan
    would invalidate the capture): defer it to the next plan creation."""
    if _capturing():
        _DEFERRED_PLANS.append((lib, handle))
        return
    lib.lars_plan_destroy(handle)


def _flush_deferred_plans():
    while _DEFERRED_PLANS and not _capturing():
        lib, handle = _DEFERRED_PLANS.pop()
        lib.lars_plan_destroy(handle)


class _Plan:
    def __init__(self, segs, nlayers, skip, grid=0, host_only=False, shared=None):
        lib = nat.load()
        _flush_deferred_plans()
        arr = (nat.Segment * max(1, len(segs)))()
        for i, (off, ln, layer, cat) in enumerate(segs):
            arr[i].offset = off
            arr[i].length = ln
            arr[i].layer = layer
            arr[i].flags = (0 if cat in skip else nat.LARS_SEG_TRUST) | \
                (nat.LARS_SEG_SHARED if shared is not None and shared[i] else 0)
        handle = nat.ctypes.c_void_p()
        flags = nat.LARS_PLAN_HOST_ONLY if host_only else 0
        nat.check(lib.lars_plan_create(arr, len(segs), nlayers, grid, flags,
                                       nat.ctypes.byref(handle)))
        self.handle = handle
        self._lib = lib
        info = nat.PlanInfo()
        nat.check(lib.lars_plan_info(handle, nat.ctypes.byref(info)))
        self.info = info
        self._finalizer = weakref.finalize(self, _destroy_plan, lib, handle)


class LarsEngine:
    """Owns the plan (per LARS skip set), the workspace and the device
    scalars (iteration counter, per-step info, per-layer sums and lambdas)
    for one FlatParamSet shard.  All launches go to the current torch
    stream."""

    def __init__(self, params):
        self.params = params
        dev = params.device
        L = len(params)
        self.nlayers = L
        self._plans = {}
        self.d_iter = torch.zeros(1, dtype=torch.int64, device=dev)
        self.d_info = torch.zeros(nat.STEP_INFO_BYTES, dtype=torch.uint8, device=dev)
        self.d_sumsq = torch.zeros(2 * L, dtype=torch.float64, device=dev)
        self.d_lambda = torch.zeros(L, dtype=torch.float64, device=dev)
        self.host_iter = 0          # value *d_iter holds after queued work
        self._ws = {}
        self._carry_version = None  # flat_param._version when the carry was written
        self._carry_key = None
        self.host_info = torch.zeros(nat.STEP_INFO_BYTES, dtype=torch.uint8).pin_memory() \
            if dev.type == "cuda" else torch.zeros(nat.STEP_INFO_BYTES, dtype=torch.uint8)

    def plan(self, skip):
        key = frozenset(skip)
        if key not in self._plans:
            segs = self.params.segments()
            p = _Plan(segs, self.nlayers, key, shared=self.params.shared_flags())
            ws = torch.empty(int(p.info.workspace_bytes), dtype=torch.uint8, device=self.params.device)
            lib = nat.load()
            nat.check(lib.lars_workspace_init(p.handle, nat.ctypes.c_void_p(ws.data_ptr()),
                                              _stream()))
            self._plans[key] = p
            self._ws[key] = ws
        return self._plans[key], self._ws[key]

    def invalidate(self):
        self._carry_version = None
        self._carry_key = None

    def carry_valid(self, key):
        return (self._carry_key == key and self._carry_version is not None
                and self._carry_version == self.params.weights_version())

    def mark_carry(self, key):
        self._carry_key = key
        self._carry_version = self.params.weights_version()

    def set_iteration(self, it):
        if it != self.host_iter:
            self.d_iter.fill_(int(it))
            self.host_iter = int(it)

    def read_info(self):
        """Blocking read of the last step's lars_step_info_t."""
        self.host_info.copy_(self.d_info, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        lr, it, bad, status = struct.unpack("<dqii", bytes(self.host_info.numpy()))
        return lr, it, bad, status

    def raise_if_diverged(self, iteration):
        _, _, bad, _ = self.read_info()
        if bad != nat.INT32_MAX:
            name = self.params.groups[bad].name
            raise DivergenceError(iteration, f"group {name} non-finite at iteration {iteration}")


def _stream():
    if torch.cuda.is_available():
        return nat.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return nat.ctypes.c_void_p(0)


def _ptr(t):
    return nat.ctypes.c_void_p(t.data_ptr())
