"""Backward-overlapped, bucketed gradient scatter for the peer-memory step.

SURVEY §8f rank 1.  The reference is strictly sequential: every worker's
backward finishes, then `all_reduce` sums the gradients (cluster.py:145-148),
then the update runs.  Here the reduce-scatter traffic moves INTO the last
micro-batch's backward:

* the flat buffer is cut into buckets of consecutive parameter groups,
  formed from the end of the buffer (backward produces the last layers'
  gradients first);
* a post-accumulate-grad hook per parameter counts the bucket down; when a
  bucket's gradient is complete (in stream order) the copy engines push, on a
  side stream, each peer's part of it straight into that peer's receive
  buffer `recv[me]` (torch SymmetricMemory, NVLink; no SM time taken from
  backward);
* the fused step (`lars_step_peer`, unchanged) then runs with its gradient
  source pointers aimed at the LOCAL receive slots instead of the peers'
  gradient buffers, so its reduce-scatter phase reads HBM, not NVLink.  The
  summation order over ranks is the same, so the result is bitwise identical
  to the non-overlapped step.

The kernel's start-of-step rank barrier is what makes the pushes safe: a rank
signals only after its own pushes completed (its step waits on the push
stream), and reuses a peer's slot only in its next backward, after the
peer's step passed its final barrier.
"""

import torch
import torch.distributed as dist

from . import _native as nat
from .errors import ProtocolError
from .flat import module_parameters


class BackwardOverlap:
    """Bucketed gradient push during the last micro-batch's backward.

    `dp` is a DataParallelLars with the "p2p" backend, `module` the torch
    module whose parameters `dp.params` was built from
    (`FlatParamSet.from_module`).  Call `arm()` right before the backward of
    the last micro-batch of a step; `dp.step()` then uses the pushed
    gradients."""

    def __init__(self, dp, module, bucket_bytes=16 << 20):
        import torch.distributed._symmetric_memory as symm_mem
        if dp.peer is None:
            raise ProtocolError("BackwardOverlap needs the 'p2p' DataParallelLars backend")
        params = dp.params
        self.dp = dp
        self.params = params
        P, C, me = params.world_size, params.shard_numel, params.rank
        dev = params.device
        mod_params = module_parameters(module)
        if len(mod_params) != len(params.groups):
            raise ProtocolError("module parameters do not match the FlatParamSet groups")
        for p, g in zip(mod_params, params.groups):
            if p.data_ptr() != g.param.data_ptr():
                raise ProtocolError(f"parameter {g.name} is not a view of the flat buffer "
                                    "(build the FlatParamSet with from_module)")
        # receive buffer: slot q holds rank q's part of this rank's shard
        self.recv = symm_mem.empty(P * C, dtype=torch.float32, device=dev)
        self.recv.zero_()
        grp = dp.coll.group or dist.group.WORLD
        h = symm_mem.rendezvous(self.recv, grp.group_name)
        off = (self.recv.data_ptr() - int(h.buffer_ptrs[h.rank])) // 4
        peer_recv = [h.get_buffer(q, (P * C,), torch.float32, off) for q in range(P)]
        # the step's peer struct, gradient sources redirected to the local slots
        s = nat.Peer.from_buffer_copy(dp.peer.struct)
        for q in range(P):
            if q != me:
                s.g_peer[q] = self.recv.data_ptr() + 4 * q * C
        self.struct = s
        # buckets of consecutive groups, from the end of the buffer
        ends = [g.offset for g in params.groups[1:]] + [params.padded_numel]
        buckets, cur, size = [], [], 0
        for i in reversed(range(len(params.groups))):
            cur.append(i)
            size += 4 * (ends[i] - params.groups[i].offset)
            if size >= bucket_bytes:
                buckets.append(cur)
                cur, size = [], 0
        if cur:
            buckets.append(cur)
        self.buckets = []
        flat_grad = params.flat_grad
        for gids in buckets:
            a, b = params.groups[min(gids)].offset, ends[max(gids)]
            copies = []
            for q in range(P):
                lo, hi = max(a, q * C), min(b, (q + 1) * C)
                if q != me and hi > lo:
                    dst = peer_recv[q][me * C + lo - q * C: me * C + hi - q * C]
                    copies.append((dst, flat_grad[lo:hi]))
            self.buckets.append((gids, copies))
        self.bucket_of = {}
        for k, (gids, _) in enumerate(self.buckets):
            for i in gids:
                self.bucket_of[i] = k
        self.stream = torch.cuda.Stream(device=dev)
        self.armed = False
        self.pending = [0] * len(self.buckets)
        self.pushed = [False] * len(self.buckets)
        self.ready = False
        self._handles = [p.register_post_accumulate_grad_hook(self._hook(i))
                         for i, p in enumerate(mod_params)]
        torch.cuda.synchronize(dev)
        dist.barrier(group=grp)

    def _hook(self, i):
        def hook(_p):
            if self.armed:
                k = self.bucket_of[i]
                self.pending[k] -= 1
                if self.pending[k] == 0:
                    self._push(k)
        return hook

    def _push(self, k):
        """Queue bucket k's pushes on the side stream after the gradient
        work queued so far on the current stream."""
        if self.pushed[k]:
            return
        self.pushed[k] = True
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            for dst, src in self.buckets[k][1]:
                dst.copy_(src, non_blocking=True)

    def arm(self):
        """Call before the backward of the last micro-batch of a step."""
        self.armed = True
        self.ready = True
        self.pending = [len(g) for g, _ in self.buckets]
        self.pushed = [False] * len(self.buckets)

    def push_all(self):
        """Queue the pushes of every bucket not pushed yet."""
        for k in range(len(self.buckets)):
            self._push(k)

    def finish(self):
        """Push whatever the hooks did not (parameters without gradient in
        this backward), make the current stream wait for every push, and
        return the peer struct for the step."""
        self.push_all()
        torch.cuda.current_stream().wait_stream(self.stream)
        self.armed = False
        self.ready = False
        return self.struct

    def remove(self):
        for hd in self._handles:
            hd.remove()
        self._handles = []
