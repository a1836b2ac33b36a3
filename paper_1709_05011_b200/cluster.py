"""Synchronous data-parallel LARS step across GPUs (one process per GPU).

Replaces the reference's in-process simulation of P workers
(pkg/src/batchlab/cluster.py):

* `all_reduce(grad_sets)` -- the reference's sum over workers with group/shape
  validation (cluster.py:124-137), for in-process lists of gradient dicts.
* `DataParallelLars` / `global_step` -- cluster.global_step minus the model
  forward/backward (cluster.py:145-156): every rank holds its local summed
  gradient in `params.flat_grad`.  Backend "p2p" (default when the buffers
  are in symmetric memory) runs the whole step as ONE kernel per rank
  (`lars_step_peer`): reduce-scatter by NVLink peer loads, per-layer sums,
  their exchange between ranks, the update, all-gather by peer stores.
  Backend "nccl" is

      reduce-scatter (NCCL, fp32 sum)     -> this rank's gradient shard
      lars_partial_norms (sm_100a kernel) -> per-layer fp64 sums of squares
      all-reduce of the [L x 2] sums      -> whole-layer norms on every rank
      lars_update (sm_100a kernel)        -> shard of w, m updated, g * 1/B
      all-gather (NCCL)                   -> every rank holds the new weights

  Either way each parameter is updated once (not once per replica as in
  cluster.py:151-153) and momentum stays sharded.  With one rank the step is
  the single fused `lars_step` launch.  `overlap_backward()` moves the
  reduce-scatter traffic into the last backward (overlap.py).
* `check_synchronized` -- replica identity check (cluster.py:101-107) over
  an on-device fingerprint, raising ConsistencyError naming the ranks.

Bitwise P-invariance of the reference's pairwise tree (reduction.py:1-10) is
not reproduced: NCCL's summation order depends on P; parity is held to the
tolerances of BASELINE.json instead.
"""

import torch
import torch.distributed as dist

from . import _native as nat
from .errors import ConsistencyError, DivergenceError, ProtocolError
from .flat import FlatParamSet, _ptr, _stream
from .optim import LambdaMap, native_hparams, scheduled_lr


def all_reduce(grad_sets):
    """cluster.py:124-137: elementwise sum over workers in the pairwise-left
    tree order (reduction.py:30-47), after validating group names / shapes."""
    ref = grad_sets[0]
    for j, g in enumerate(grad_sets[1:], start=1):
        if set(g) != set(ref):
            raise ProtocolError(f"worker {j} gradient groups differ from worker 0")
        for name in ref:
            if tuple(g[name].shape) != tuple(ref[name].shape):
                raise ProtocolError(f"shape mismatch in group {name!r} on worker {j}")
    items = list(grad_sets)
    while len(items) > 1:
        nxt = [{k: items[i][k] + items[i + 1][k] for k in items[i]}
               for i in range(0, len(items) - 1, 2)]
        if len(items) % 2:
            nxt.append(items[-1])
        items = nxt
    return items[0]


class NativeKernels:
    """The two halves of the split LARS step, through liblars_b200.so."""

    def partial_norms(self, eng, plan, ws, w_shard, g_shard, h):
        nat.check(nat.load().lars_partial_norms(
            plan.handle, _ptr(w_shard), _ptr(g_shard), nat.ctypes.byref(h), _ptr(eng.d_iter),
            _ptr(eng.d_sumsq), _ptr(eng.d_info), _ptr(ws), _stream()))

    def update(self, eng, plan, ws, w_shard, g_shard, m_shard, h):
        nat.check(nat.load().lars_update(
            plan.handle, _ptr(w_shard), _ptr(g_shard), _ptr(m_shard), nat.ctypes.byref(h),
            _ptr(eng.d_sumsq), _ptr(eng.d_lambda), _ptr(eng.d_info), _ptr(ws), _stream()))


class Collectives:
    """reduce-scatter / all-reduce / all-gather on a process group.  NCCL
    does each in one call; backends without the tensor forms (gloo) go
    through all_reduce / all_gather lists."""

    def __init__(self, group=None):
        self.group = group
        self.backend = dist.get_backend(group)

    def reduce_scatter(self, out, inp):
        if self.backend == "nccl":
            dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=self.group)
        else:
            tmp = inp.clone()
            dist.all_reduce(tmp, group=self.group)
            r, n = dist.get_rank(self.group), out.numel()
            out.copy_(tmp[r * n:(r + 1) * n])

    def all_reduce(self, t):
        dist.all_reduce(t, group=self.group)

    def all_gather(self, out, inp):
        if self.backend == "nccl":
            dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            parts = list(out.chunk(dist.get_world_size(self.group)))
            dist.all_gather(parts, inp.clone(), group=self.group)


class _PeerState:
    """Peer pointers (torch SymmetricMemory) of the fused peer-memory step."""

    def __init__(self, params, group):
        import torch.distributed._symmetric_memory as symm_mem
        if not params.symmetric:
            raise ProtocolError("backend='p2p' needs FlatParamSet(..., symmetric=True)")
        P, L = params.world_size, len(params)
        if P > nat.MAX_RANKS:
            raise ProtocolError(f"backend='p2p' supports up to {nat.MAX_RANKS} ranks")
        grp = group or dist.group.WORLD
        name = grp.group_name
        dev = params.device
        # norm exchange: [P][L][2] for lars_step_peer; two regions of [P] rows
        # of 2L+2 (values + tag) for lars_step_peer_stream
        self.xnorm = symm_mem.empty(2 * P * (2 * L + 2), dtype=torch.float64, device=dev)
        self.flags = symm_mem.empty(max(P, 4), dtype=torch.int32, device=dev)
        self.xnorm.zero_()
        self.flags.zero_()
        self.g_shard = torch.zeros(params.shard_numel, dtype=torch.float32, device=dev)

        def peers(t):
            h = symm_mem.rendezvous(t, name)
            delta = t.data_ptr() - int(h.buffer_ptrs[h.rank])
            return [int(p) + delta for p in h.buffer_ptrs]

        s = nat.Peer()
        lo4 = 4 * params.shard_lo
        for q, (w, g, x, f) in enumerate(zip(peers(params.flat_param), peers(params.flat_grad),
                                             peers(self.xnorm), peers(self.flags))):
            s.w_peer[q] = w + lo4
            s.g_peer[q] = g + lo4
            s.x_peer[q] = x
            s.f_peer[q] = f
        s.g_shard = self.g_shard.data_ptr()
        s.m = params.momentum.data_ptr()
        s.rank = params.rank
        s.world = P
        self.struct = s
        torch.cuda.synchronize(dev)
        dist.barrier(group=grp)


class DataParallelLars:
    """The sharded RS -> LARS -> AG step for one FlatParamSet shard.

    backend "nccl": NCCL reduce-scatter / all-reduce / all-gather around the
    split kernels.  backend "p2p": ONE fused kernel per rank doing the
    reduce-scatter (peer loads), the norm exchange, the update and the
    all-gather (peer stores) over NVLink peer memory; needs a
    FlatParamSet(symmetric=True).  backend "p2p-stream": the same step with
    the reduce-scatter and the update + all-gather pipelined over the shard's
    segments (`lars_step_peer_stream`: inbound and outbound NVLink traffic
    overlap).  "auto" picks "p2p" when possible."""

    def __init__(self, params, group=None, kernels=None, backend="auto"):
        if not isinstance(params, FlatParamSet):
            raise TypeError("DataParallelLars needs a FlatParamSet")
        self.params = params
        self.coll_group = group
        self.P = params.world_size
        self.kernels = kernels or NativeKernels()
        self.peer = None
        self.overlap = None
        self.backend = "local" if self.P == 1 else backend
        if self.P > 1:
            if dist.get_world_size(group) != self.P or dist.get_rank(group) != params.rank:
                raise ProtocolError("FlatParamSet world/rank do not match the process group")
            self.coll = Collectives(group)
            if backend in ("auto", "p2p", "p2p-stream") and kernels is None and params.symmetric:
                try:
                    self.peer = _PeerState(params, group)
                    self.backend = "p2p" if backend == "auto" else backend
                except Exception:
                    if backend != "auto":
                        raise
            if backend in ("p2p", "p2p-stream") and self.peer is None:
                raise ProtocolError(f"backend={backend!r} needs a symmetric FlatParamSet")
            if self.peer is None:
                self.backend = "nccl"
                self.g_shard = torch.zeros(params.shard_numel, dtype=torch.float32,
                                           device=params.device)
        else:
            self.coll = None
            self.g_shard = None

    def overlap_backward(self, module, bucket_bytes=16 << 20):
        """Push gradient buckets to their owners during the last micro-batch's
        backward (overlap.BackwardOverlap; "p2p" backend only).  Call
        `.arm()` on the returned object before that backward."""
        from .overlap import BackwardOverlap
        self.overlap = BackwardOverlap(self, module, bucket_bytes)
        return self.overlap

    def _prepare(self, hp, st, *, grad_scale, lr, carry=None):
        """Host-side checks and the packed hparams of one step."""
        if lr is None:
            scheduled_lr(hp, st)  # ScheduleExhaustedError before launching (optim.py:84-87)
        eng = self.params.engine()
        key = frozenset(hp.lars_skip_categories)
        plan, ws = eng.plan(key)
        flags = 0
        if lr is None:
            eng.set_iteration(st.iteration)
            flags |= nat.LARS_STEP_ADVANCE_ITER
        if carry if carry is not None else eng.carry_valid(key):
            flags |= nat.LARS_STEP_USE_WCARRY
        h = native_hparams(hp, st, lr=lr, grad_scale=grad_scale, flags=flags)
        return eng, key, plan, ws, h

    def _enqueue(self, eng, plan, ws, h, timers=None):
        """Queue the whole step on the current stream (graph-capturable)."""
        params = self.params
        rec = (lambda name: timers.append((name, _event()))) if timers is not None else (lambda n: None)
        if self.P == 1:
            rec("start")
            nat.check(nat.load().lars_step(
                plan.handle, _ptr(params.flat_param), _ptr(params.flat_grad),
                _ptr(params.momentum), nat.ctypes.byref(h), _ptr(eng.d_iter), _ptr(eng.d_sumsq),
                _ptr(eng.d_lambda), _ptr(eng.d_info), _ptr(ws), _stream()))
            rec("lars_step")
            return
        if self.peer is not None:
            # gradients pushed during backward (overlap.py): reduce from the
            # local receive slots instead of over NVLink
            ov = self.overlap
            struct = ov.finish() if ov is not None and ov.ready else self.peer.struct
            rec("start")
            fn = nat.load().lars_step_peer_stream if self.backend == "p2p-stream" \
                else nat.load().lars_step_peer
            nat.check(fn(plan.handle, nat.ctypes.byref(struct), nat.ctypes.byref(h),
                         _ptr(eng.d_iter), _ptr(eng.d_sumsq), _ptr(eng.d_lambda), _ptr(eng.d_info),
                         _ptr(ws), _stream()))
            rec("lars_step_peer_stream" if self.backend == "p2p-stream" else "lars_step_peer")
            return
        w_shard = params.param_shard
        rec("start")
        self.coll.reduce_scatter(self.g_shard, params.flat_grad)
        rec("reduce_scatter")
        self.kernels.partial_norms(eng, plan, ws, w_shard, self.g_shard, h)
        rec("partial_norms")
        self.coll.all_reduce(eng.d_sumsq)
        rec("norm_all_reduce")
        self.kernels.update(eng, plan, ws, w_shard, self.g_shard, params.momentum, h)
        rec("update")
        self.coll.all_gather(params.flat_param, w_shard)
        rec("all_gather")

    def step(self, hp, st, *, grad_scale=1.0, lr=None, check=False, timers=None):
        """One synchronous step.  `st` advances like sgd_step (unless an
        explicit `lr` is given: the apply_update form, st untouched).
        Returns the lambdas (lazy mapping).  `timers`, if a list, receives
        (phase, cuda event) pairs recorded on the current stream."""
        iteration = st.iteration if st is not None else 0
        eng, key, plan, ws, h = self._prepare(hp, st, grad_scale=grad_scale, lr=lr)
        self._enqueue(eng, plan, ws, h, timers)
        eng.mark_carry(key)
        if lr is None:
            eng.host_iter = iteration + 1
        lams = LambdaMap(self.params.names(), eng.d_lambda.clone())
        if check:
            self.raise_if_diverged(iteration)
        if lr is None:
            st.iteration += 1
        return lams

    def capture(self, hp, st, *, grad_scale=1.0):
        """Capture the scheduled step (device lr, device iteration counter,
        carried ||w||) into a CUDA graph.  Call after at least one eager
        step.  Returns a GraphedStep whose replay() advances `st`.

        The graph bakes in the carried ||w||^2 (phase A reads only g), so the
        carry must be valid now -- i.e. an eager step ran since the weights
        were last written -- and `replay()` falls back to one eager step
        whenever a write since the last step invalidated it."""
        key = frozenset(hp.lars_skip_categories)
        if not self.params.engine().carry_valid(key):
            raise ProtocolError("capture() needs a valid norm carry: run one eager step() after "
                                "the weights were last written")
        eng, key, plan, ws, h = self._prepare(hp, st, grad_scale=grad_scale, lr=None, carry=True)
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                self._enqueue(eng, plan, ws, h)
        torch.cuda.current_stream().wait_stream(side)
        return GraphedStep(self, graph, hp, st, key, grad_scale)

    def align(self, hp):
        """Device-side cross-rank barrier on the current stream (no host
        sync): every rank leaves it at the same time.  For benchmarks that
        put untimed, per-GPU-variable work (an L2 flush) before a timed
        step.  Every rank must call it the same number of times."""
        if self.P == 1:
            return
        if self.peer is not None:
            eng = self.params.engine()
            _, ws = eng.plan(frozenset(hp.lars_skip_categories))
            nat.check(nat.load().lars_peer_barrier(nat.ctypes.byref(self.peer.struct), _ptr(ws),
                                                   _ptr(eng.d_info), _stream()))
        else:
            t = torch.zeros(1, device=self.params.device)
            self.coll.all_reduce(t)

    def raise_if_diverged(self, iteration):
        """DivergenceError(iteration) if any rank's last step produced
        non-finite weights (the first such group in order); ProtocolError if
        a cross-rank barrier of the peer kernel timed out."""
        eng = self.params.engine()
        v = eng.d_info.view(torch.int32)[4:6].clone()   # nonfinite_layer, status
        v[1] = -v[1]
        if self.coll is not None:
            dist.all_reduce(v, op=dist.ReduceOp.MIN, group=self.coll.group)
        b, status = int(v[0].item()), -int(v[1].item())
        if status & nat.LARS_STATUS_RANK_TIMEOUT:
            raise ProtocolError("a peer rank did not reach the step's cross-rank barrier within "
                                "60 s; the step's results are invalid")
        if b != nat.INT32_MAX:
            name = self.params.groups[b].name
            raise DivergenceError(iteration, f"group {name} non-finite at iteration {iteration}")


class GraphedStep:
    """Replays a captured DP step; keeps the host ScheduleState in step with
    the device counter and refuses an exhausted schedule on the host."""

    def __init__(self, dp, graph, hp, st, key, grad_scale):
        self.dp, self.graph, self.hp, self.st, self.key = dp, graph, hp, st, key
        self.grad_scale = grad_scale

    def replay(self):
        """One scheduled step.  If the weights were written since the last
        step (checkpoint restore, load_state_dict, in-place averaging) the
        captured carry is stale: run the step eagerly with fresh norms
        instead (same result, one more launch), which re-validates it."""
        eng = self.dp.params.engine()
        if not eng.carry_valid(self.key):
            self.dp.step(self.hp, self.st, grad_scale=self.grad_scale)
            return
        scheduled_lr(self.hp, self.st)
        eng.set_iteration(self.st.iteration)
        self.graph.replay()
        eng.mark_carry(self.key)
        eng.host_iter = self.st.iteration + 1
        self.st.iteration += 1

    def lambdas(self):
        eng = self.dp.params.engine()
        return LambdaMap(self.dp.params.names(), eng.d_lambda.clone())


def _event():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def global_step(params, hp, st, global_batch, *, group=None, check=True):
    """cluster.global_step (cluster.py:145-156) after the local backward:
    sum the ranks' gradients, divide by the global batch, update once, and
    leave every rank with the same weights.  Returns the lambdas.  The
    DataParallelLars lives on the FlatParamSet (freed with it)."""
    dp = getattr(params, "_dp", None)
    if dp is None or dp.coll_group is not group:
        dp = params._dp = DataParallelLars(params, group)
    return dp.step(hp, st, grad_scale=1.0 / global_batch, check=check)


def check_synchronized(params, group=None):
    """cluster.py:101-107 across ranks: all ranks must hold identical weights."""
    if params.world_size == 1 or not dist.is_initialized():
        return
    fp = params.fingerprint()
    allfp = [torch.zeros_like(fp) for _ in range(dist.get_world_size(group))]
    dist.all_gather(allfp, fp, group=group)
    bad = [r for r, f in enumerate(allfp) if not torch.equal(f, allfp[0])]
    if bad:
        raise ConsistencyError(f"replicas desynchronized: ranks {bad} differ from rank 0")
