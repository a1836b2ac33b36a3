"""Host-resident (reference-style numpy) parameter sets on the device step.

The reference's ParamSet (pkg/src/batchlab/nn.py:72-114) holds one
caller-owned fp64 array per group for `param`, `grad` and `momentum_buf`, and
optim.apply_update (optim.py:117-134) mutates `param` and `momentum_buf` in
place.  `HostMirror` runs that call on the device step without host-side
packing or conversion:

* arrays of at least REGISTER_MIN_BYTES are pinned where they lie
  (`lars_host_register`, once; the mirror keeps them alive while pinned) and
  DMA'd straight from / into the caller's memory; smaller ones (and any array
  that cannot be pinned, e.g. one sharing pages with a pinned one) go through
  one pinned bounce buffer;
* fp64 <-> fp32 conversion of the flat buffers runs on the device
  (`lars_host_copy_in` / `lars_host_copy_out`: the DMAs plus one conversion
  launch per buffer);
* after the step the first non-finite group is read back before anything is
  written to the host, and only the groups up to and including it are
  written back -- the state the reference leaves when apply_update raises
  DivergenceError (optim.py:125-133).
"""

import weakref

import numpy as np
import torch

from . import _native as nat
from .flat import FlatParamSet, _ptr, _stream

REGISTER_MIN_BYTES = 1 << 20
_ATTRS = ("param", "grad", "momentum_buf")


def _unregister_all(lib, registered):
    for ptr in list(registered):
        lib.lars_host_unregister(nat.ctypes.c_void_p(ptr))
    registered.clear()


class HostMirror:
    """Device mirror of one reference-style ParamSet (same group order)."""

    def __init__(self, groups, device=None):
        groups = list(groups)
        layout = [(g.name, tuple(np.shape(g.param)), g.category) for g in groups]
        self.fps = FlatParamSet(layout, device)
        self.names = [g.name for g in groups]
        self.signature = _signature(groups)
        dev = self.fps.device
        self.stage = torch.zeros(self.fps.padded_numel, dtype=torch.float64, device=dev)
        # bounce buffer: one fp64 region per (array kind, small group)
        small = [g for g in self.fps.groups if 8 * g.numel < REGISTER_MIN_BYTES]
        total = sum(g.numel for g in small)
        host = torch.empty(max(1, 3 * total), dtype=torch.float64, pin_memory=dev.type == "cuda")
        self._bounce_host = host
        flat = host.numpy()
        self._bounce = [dict() for _ in _ATTRS]
        off = 0
        for k in range(len(_ATTRS)):
            for g in small:
                self._bounce[k][g.index] = flat[off:off + g.numel]
                off += g.numel
        self._lib = nat.load()
        self._registered = {}  # host pointer -> (array kept alive, bytes)
        self._finalizer = weakref.finalize(self, _unregister_all, self._lib, self._registered)

    # ---- pinning ------------------------------------------------------------
    def _pinned_ptr(self, arr):
        """Pointer usable for DMA of `arr` in place, or None."""
        if (not isinstance(arr, np.ndarray) or arr.dtype != np.float64
                or not arr.flags.c_contiguous or arr.nbytes < REGISTER_MIN_BYTES):
            return None
        ptr = arr.ctypes.data
        have = self._registered.get(ptr)
        if have is not None and have[1] == arr.nbytes:
            return ptr
        if have is not None:                        # same start, other extent
            self._lib.lars_host_unregister(nat.ctypes.c_void_p(ptr))
            del self._registered[ptr]
        rc = self._lib.lars_host_register(nat.ctypes.c_void_p(ptr), arr.nbytes)
        if rc != nat.LARS_OK:
            if rc != nat.LARS_ERR_HOST_MEMORY:
                nat.check(rc)
            return None
        self._registered[ptr] = (arr, arr.nbytes)
        return ptr

    def _release_stale(self, live):
        for ptr in [p for p in self._registered if p not in live]:
            self._lib.lars_host_unregister(nat.ctypes.c_void_p(ptr))
            del self._registered[ptr]

    def _spans(self, groups, k, upto=None, live=None):
        """Span table of array kind k (param / grad / momentum_buf) and the
        (bounce view, caller array) pairs that go through the bounce buffer."""
        n = len(groups) if upto is None else upto
        spans = (nat.HostSpan * max(1, n))()
        bounced = []
        for i in range(n):
            src, dst = groups[i], self.fps.groups[i]
            arr = getattr(src, _ATTRS[k])
            if np.size(arr) != dst.numel:  # DMA sizes come from the mirror's layout
                raise ValueError(f"group {dst.name}: {_ATTRS[k]} has {np.size(arr)} elements, "
                                 f"expected {dst.numel}")
            ptr = self._pinned_ptr(arr)
            if ptr is None:
                view = self._bounce[k].get(i)
                if view is None:  # a big array that could not be pinned in place
                    view = self._bounce[k][i] = torch.empty(
                        dst.numel, dtype=torch.float64, pin_memory=True).numpy()
                bounced.append((view, arr))
                ptr = view.ctypes.data
            elif live is not None:
                live.add(ptr)
            spans[i].host = ptr
            spans[i].offset = dst.offset
            spans[i].numel = dst.numel
        return spans, n, bounced

    # ---- copies -------------------------------------------------------------
    def load(self, groups):
        """Caller arrays -> flat fp32 device buffers (async on the current stream)."""
        if _signature(groups) != self.signature:
            raise ValueError("parameter groups changed since the mirror was built")
        live = set()
        dsts = (self.fps.flat_param, self.fps.flat_grad, self.fps.momentum)
        for k, dst in enumerate(dsts):
            spans, n, bounced = self._spans(groups, k, live=live)
            for view, arr in bounced:
                np.copyto(view, np.reshape(arr, -1), casting="unsafe")
            nat.check(self._lib.lars_host_copy_in(spans, n, _ptr(self.stage), _ptr(dst),
                                                  self.fps.padded_numel, _stream()))
        self._release_stale(live)
        self.fps.invalidate_norm_cache()

    def store(self, groups, upto=None):
        """Flat device w and m -> caller's `param` / `momentum_buf` arrays for
        the first `upto` groups (all if None); returns after the copies landed."""
        pending = []
        # (the stage buffer is reused by the second conversion: stream order
        # puts it after the first one's D2H)
        for k, src in ((0, self.fps.flat_param), (2, self.fps.momentum)):
            spans, n, bounced = self._spans(groups, k, upto=upto)
            nat.check(self._lib.lars_host_copy_out(_ptr(src), _ptr(self.stage),
                                                   self.fps.padded_numel, spans, n, _stream()))
            pending.extend(bounced)
        torch.cuda.current_stream().synchronize()
        for view, arr in pending:
            np.copyto(arr, view.reshape(np.shape(arr)), casting="unsafe")


def _signature(groups):
    return [(g.name, tuple(np.shape(g.param)), g.category) for g in groups]


_mirrors = weakref.WeakKeyDictionary()


def mirror_for(params, device=None):
    """The HostMirror of a reference-style ParamSet (built on first use,
    rebuilt if its groups' names, shapes or categories changed; freed with
    the ParamSet)."""
    groups = list(params)
    try:
        m = _mirrors.get(params)
    except TypeError:
        m = None
    if m is None or m.signature != _signature(groups):
        m = HostMirror(groups, device)
        try:
            _mirrors[params] = m
        except TypeError:
            pass
    return m, groups


def mirror_of(params):
    """The existing mirror of `params`, or None."""
    try:
        return _mirrors.get(params)
    except TypeError:
        return None
