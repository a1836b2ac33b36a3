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
* the groups are split into contiguous parts of at least PART_MIN_ELEMS
  elements (at most MAX_PARTS), each with its own flat buffers and step
  plan: a layer's update needs only its own norms, so part i's weights and
  momentum go back to the host (PCIe device-to-host) while part i+1's
  arrays are still coming in (host-to-device) -- the two directions of the
  link overlap instead of running one after the other;
* before a part is written back its first non-finite group is read, and only
  the groups up to and including it are written, nothing after -- the state
  the reference leaves when apply_update raises DivergenceError
  (optim.py:125-133).
"""

import struct
import weakref

import numpy as np
import torch

from . import _native as nat
from .flat import FlatParamSet, _ptr, _stream

REGISTER_MIN_BYTES = 1 << 20
PART_MIN_ELEMS = 4 << 20   # pipeline granularity (a part is a run of whole groups)
MAX_PARTS = 8
_ATTRS = ("param", "grad", "momentum_buf")


def _unregister_all(lib, registered):
    for ptr in list(registered):
        lib.lars_host_unregister(nat.ctypes.c_void_p(ptr))
    registered.clear()


def _split(numels, min_elems, max_parts):
    """Contiguous group ranges [(g0, g1)] of roughly equal element counts."""
    total = sum(numels)
    k = max(1, min(max_parts, total // max(1, min_elems), len(numels)))
    target = total / k
    parts, g0, acc = [], 0, 0
    for i, n in enumerate(numels):
        acc += n
        if acc >= target * (len(parts) + 1) and len(parts) < k - 1 and i + 1 < len(numels):
            parts.append((g0, i + 1))
            g0 = i + 1
    parts.append((g0, len(numels)))
    return parts


class _Part:
    """One contiguous run of groups: flat buffers, plan, fp64 staging."""

    def __init__(self, layout, g0, g1, device):
        self.g0, self.g1 = g0, g1
        self.fps = FlatParamSet(layout[g0:g1], device)
        # fp64 staging per array kind, so every kind's DMAs can be in flight
        self.stage = [torch.zeros(self.fps.padded_numel, dtype=torch.float64, device=self.fps.device)
                      for _ in _ATTRS]
        self.done = None  # event: this part's step finished (and its info copied)


class HostMirror:
    """Device mirror of one reference-style ParamSet (same group order)."""

    def __init__(self, groups, device=None):
        groups = list(groups)
        layout = [(g.name, tuple(np.shape(g.param)), g.category) for g in groups]
        self.names = [g.name for g in groups]
        self.signature = _signature(groups)
        numels = [int(np.prod(s)) for _, s, _ in layout]
        self.parts = [_Part(layout, g0, g1, device)
                      for g0, g1 in _split(numels, PART_MIN_ELEMS, MAX_PARTS)]
        dev = self.parts[0].fps.device
        self.device = dev
        self.last_bad = None  # global index of the last step's first non-finite group
        # bounce buffer for the small groups: per part, runs of consecutive
        # small groups laid out exactly like the part's staging buffer
        # (padding included, left zero), so one DMA moves a whole run; one
        # fp64 region per (array kind, run)
        self._small = [8 * n < REGISTER_MIN_BYTES for n in numels]
        self._runs = []   # per part: [(g_a, g_b, stage offset, length)]
        total = 0
        for part in self.parts:
            runs, j = [], part.g0
            while j < part.g1:
                if not self._small[j]:
                    j += 1
                    continue
                a = j
                while j < part.g1 and self._small[j]:
                    j += 1
                ga, gb = part.fps.groups[a - part.g0], part.fps.groups[j - 1 - part.g0]
                runs.append((a, j, ga.offset, gb.offset + gb.numel - ga.offset))
                total += runs[-1][3]
            self._runs.append(runs)
        host = torch.zeros(max(1, 3 * total), dtype=torch.float64, pin_memory=dev.type == "cuda")
        self._bounce_host = host
        flat = host.numpy()
        self._runbuf = [dict() for _ in _ATTRS]   # (g_a) -> run buffer
        self._bounce = [dict() for _ in _ATTRS]   # group -> its view (runs, or a big unpinnable array)
        off = 0
        for k in range(len(_ATTRS)):
            for pi, part in enumerate(self.parts):
                for a, b, o0, ln in self._runs[pi]:
                    buf = flat[off:off + ln]
                    off += ln
                    self._runbuf[k][a] = buf
                    for i in range(a, b):
                        g = part.fps.groups[i - part.g0]
                        self._bounce[k][i] = buf[g.offset - o0:g.offset - o0 + g.numel]
        self._lib = nat.load()
        self._registered = {}  # host pointer -> (array kept alive, bytes)
        self._finalizer = weakref.finalize(self, _unregister_all, self._lib, self._registered)
        if dev.type == "cuda":
            self._s_in = torch.cuda.Stream(dev)
            self._s_out = torch.cuda.Stream(dev)

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

    def _spans(self, groups, k, part, upto=None, live=None, which=None):
        """Span table of array kind k (param / grad / momentum_buf) for the
        groups of `part` (global indices below `upto`, if given) and the
        (bounce view, caller array) pairs that go through the bounce buffer.
        `which`: None for every group, "pinned" / "bounced" for one kind."""
        g1 = part.g1 if upto is None else min(part.g1, upto)
        n = 0
        spans = (nat.HostSpan * max(1, g1 - part.g0))()
        bounced = []
        if which != "pinned":  # runs of small groups: one span each
            for a, b, o0, ln in self._runs[self.parts.index(part)]:
                if a >= g1:
                    break
                last = part.fps.groups[min(b, g1) - 1 - part.g0]
                for i in range(a, min(b, g1)):
                    arr = getattr(groups[i], _ATTRS[k])
                    numel = part.fps.groups[i - part.g0].numel
                    if np.size(arr) != numel:
                        raise ValueError(f"group {self.names[i]}: {_ATTRS[k]} has {np.size(arr)} "
                                         f"elements, expected {numel}")
                    bounced.append((self._bounce[k][i], arr))
                spans[n].host = self._runbuf[k][a].ctypes.data
                spans[n].offset = o0
                spans[n].numel = last.offset + last.numel - o0
                n += 1
        for j in range(max(0, g1 - part.g0)):
            i = part.g0 + j
            if self._small[i]:
                continue
            dst = part.fps.groups[j]
            arr = getattr(groups[i], _ATTRS[k])
            if np.size(arr) != dst.numel:  # DMA sizes come from the mirror's layout
                raise ValueError(f"group {dst.name}: {_ATTRS[k]} has {np.size(arr)} elements, "
                                 f"expected {dst.numel}")
            ptr = self._pinned_ptr(arr)
            if ptr is None:
                if which == "pinned":
                    continue
                view = self._bounce[k].get(i)
                if view is None:  # a big array that could not be pinned in place
                    view = self._bounce[k][i] = torch.empty(
                        dst.numel, dtype=torch.float64, pin_memory=True).numpy()
                bounced.append((view, arr))
                ptr = view.ctypes.data
            else:
                if which == "bounced":
                    continue
                if live is not None:
                    live.add(ptr)
            spans[n].host = ptr
            spans[n].offset = dst.offset
            spans[n].numel = dst.numel
            n += 1
        return spans, n, bounced

    # ---- copies -------------------------------------------------------------
    def _load_part(self, groups, part, live):
        """Caller arrays of `part` -> its flat fp32 buffers (current stream).
        The DMAs of the arrays pinned in place are queued first, so the
        device moves them while the host fills the bounce buffer for the
        small ones; each copy-in converts its staging buffer (the second
        conversion of a kind rewrites the first one's stale small groups)."""
        fps = part.fps
        dsts = (fps.flat_param, fps.flat_grad, fps.momentum)
        for which in ("pinned", "bounced"):
            for k, dst in enumerate(dsts):
                spans, n, bounced = self._spans(groups, k, part, live=live, which=which)
                if n == 0:
                    continue
                for view, arr in bounced:
                    np.copyto(view, np.reshape(arr, -1), casting="unsafe")
                nat.check(self._lib.lars_host_copy_in(spans, n, _ptr(part.stage[k]), _ptr(dst),
                                                      fps.padded_numel, _stream()))
        fps.invalidate_norm_cache()

    def _store_part(self, groups, part, upto=None):
        """Flat device w and m of `part` -> the caller's `param` /
        `momentum_buf` (groups below `upto`), on the current stream; returns
        the bounced pairs to copy once the stream is done."""
        pending = []
        for k, src in ((0, part.fps.flat_param), (2, part.fps.momentum)):
            spans, n, bounced = self._spans(groups, k, part, upto=upto)
            if n == 0:
                continue
            nat.check(self._lib.lars_host_copy_out(_ptr(src), _ptr(part.stage[k]),
                                                   part.fps.padded_numel, spans, n, _stream()))
            pending.extend(bounced)
        return pending

    def step(self, groups, hp, lr, iteration, grad_scale, check, launch):
        """One apply_update over the caller's arrays: per part, copy in and
        step (`launch(fps)` enqueues the step on the current stream); write
        each part back as soon as its step is done, stopping after the first
        non-finite group when `check`.  Returns (lambdas by name, global
        index of the first non-finite group or None)."""
        if _signature(groups) != self.signature:
            raise ValueError("parameter groups changed since the mirror was built")
        live = set()
        if self.device.type != "cuda":
            raise RuntimeError("host parameter sets need the CUDA device path")
        main = torch.cuda.current_stream(self.device)
        self._s_in.wait_stream(main)
        with torch.cuda.stream(self._s_in):
            for part in self.parts:
                self._load_part(groups, part, live)
                launch(part.fps)
                part.done = torch.cuda.Event()
                part.done.record(self._s_in)
        self._release_stale(live)
        pending, bad = [], None
        with torch.cuda.stream(self._s_out):
            for part in self.parts:
                # the step's status word comes back on the write-back stream:
                # a device-to-host copy queued on the copy-in stream would
                # wait behind the previous part's write-back on the same copy
                # engine and stall every later copy-in
                eng = part.fps.engine()
                self._s_out.wait_event(part.done)
                eng.host_info.copy_(eng.d_info, non_blocking=True)
                info_ready = torch.cuda.Event()
                info_ready.record(self._s_out)
                info_ready.synchronize()
                _, _, local_bad, _ = struct.unpack("<dqii", bytes(eng.host_info.numpy()))
                if local_bad != nat.INT32_MAX:
                    bad = part.g0 + local_bad
                    if check:
                        pending.extend(self._store_part(groups, part, upto=bad + 1))
                        break
                pending.extend(self._store_part(groups, part))
        self._s_out.synchronize()
        for view, arr in pending:
            np.copyto(arr, view.reshape(np.shape(arr)), casting="unsafe")
        main.wait_stream(self._s_out)
        main.wait_stream(self._s_in)  # (parts after a divergence were not waited for)
        lam = torch.cat([p.fps.engine().d_lambda for p in self.parts]).cpu().tolist()
        self.last_bad = bad
        return dict(zip(self.names, lam)), bad


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
