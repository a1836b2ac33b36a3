"""CPU oracle for the LARS data-parallel step -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy fp64 restatement of the reference's hot path.  It
is the parity checker for the CUDA path and the timed CPU baseline in
`bench.py`; nothing in `paper_1709_05011_b200/` imports it and the product path
never routes through it (only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may use it).

Parity pinning: `tests/test_oracle.py` checks every function here against the
reference's own known-answer tests (`pkg/tests/test_optim.py:17-222`,
`pkg/tests/test_cluster.py:93-105`, `pkg/tests/test_acceptance.py:166-182`,
restated) and against golden vectors produced by running the reference itself
in the build container (`tests/golden/make_golden.py`, which imports
`/root/reference/pkg/src/batchlab`; the vectors are committed under
`tests/golden/`).

Evaluation order follows the reference line by line; each function cites the
lines it restates.  Hyperparameters are duck-typed: any object with the
reference `HyperParams` attribute names (`optim.py:25-36`) works.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np

WEIGHT = "weight"            # nn.py:33
BIAS = "bias"                # nn.py:34
NORM_SCALE = "norm-scale"    # nn.py:35
NORM_SHIFT = "norm-shift"    # nn.py:36
DEFAULT_LARS_SKIP = frozenset({BIAS, NORM_SCALE, NORM_SHIFT})  # optim.py:22


class OracleScheduleExhausted(Exception):
    """Stands in for ScheduleExhaustedError (optim.py:84-87)."""


class OracleDivergence(Exception):
    """Stands in for DivergenceError(iteration) (optim.py:132-133)."""

    def __init__(self, iteration, group):
        self.iteration = iteration
        self.group = group
        super().__init__(f"group {group} non-finite at iteration {iteration}")


class Group:
    """One parameter group: the fields of `nn.ParamGroup` (nn.py:63-69)."""

    __slots__ = ("name", "param", "grad", "momentum_buf", "category")

    def __init__(self, name, param, grad, momentum_buf, category):
        self.name = name
        self.param = param
        self.grad = grad
        self.momentum_buf = momentum_buf
        self.category = category

    def copy(self):
        return Group(self.name, self.param.copy(), self.grad.copy(),
                     self.momentum_buf.copy(), self.category)


def linear_scaled_lr(base_lr, base_batch, new_batch):
    """optim.py:69-73."""
    if base_batch <= 0 or new_batch <= 0:
        raise ValueError("batch sizes must be positive")
    return base_lr * (new_batch / base_batch)


def max_iterations(epochs, n, batch_size):
    """optim.py:145-147: floor(E * n / B)."""
    return (epochs * n) // batch_size


def scheduled_lr(hp, iteration, max_iters, iters_per_epoch):
    """optim.py:76-95, same operand order (Python evaluates left to right)."""
    it = iteration
    if it > max_iters:                                           # :84
        raise OracleScheduleExhausted(f"iteration {it} past schedule end {max_iters}")
    warmup_iters = hp.warmup_epochs * iters_per_epoch            # :88
    if it < warmup_iters:                                        # :89
        return hp.base_lr * (it + 1) / warmup_iters              # :90
    span = max_iters - warmup_iters                              # :91
    if span <= 0:                                                # :92
        return 0.0                                               # :93
    progress = (it - warmup_iters) / span                        # :94
    return hp.base_lr * (1.0 - progress) ** hp.poly_power        # :95


def lars_local_lr(param, grad, weight_decay, trust):
    """optim.py:98-108.  ||x|| is numpy's 2-norm (a BLAS ddot + sqrt for fp64)."""
    w_norm = float(np.linalg.norm(param))                        # :100
    g_norm = float(np.linalg.norm(grad))                         # :101
    denom = g_norm + weight_decay * w_norm                       # :102
    if w_norm == 0.0:                                            # :103
        return 0.0                                               # :104
    if denom == 0.0:                                             # :105
        return 1.0                                               # :107
    return trust * w_norm / denom                                # :108


def lars_from_sumsq(w_sumsq, g_sumsq, weight_decay, trust):
    """optim.py:98-108 with the two squared norms already reduced."""
    w_norm = float(np.sqrt(w_sumsq))
    g_norm = float(np.sqrt(g_sumsq))
    denom = g_norm + weight_decay * w_norm
    if w_norm == 0.0:
        return 0.0
    if denom == 0.0:
        return 1.0
    return trust * w_norm / denom


def group_local_lr(group, hp):
    """optim.py:111-114."""
    if not hp.lars_enabled or group.category in hp.lars_skip_categories:
        return 1.0
    return lars_local_lr(group.param, group.grad, hp.weight_decay, hp.lars_trust)


def apply_update(groups, hp, lr, iteration=0):
    """optim.py:117-134: per group in order, lambda, coupled WD, momentum with
    the LR inside it, write-back, then the non-finite check after that group."""
    lambdas = {}
    for g in groups:                                             # :125
        lam = group_local_lr(g, hp)                              # :126
        lambdas[g.name] = lam                                    # :127
        step_g = g.grad + hp.weight_decay * g.param              # :128
        g.momentum_buf *= hp.momentum                            # :129
        g.momentum_buf += (lam * lr) * step_g                    # :130
        g.param -= g.momentum_buf                                # :131
        if not np.all(np.isfinite(g.param)):                     # :132
            raise OracleDivergence(iteration, g.name)            # :133
    return lambdas


def sgd_step(groups, hp, iteration, max_iters, iters_per_epoch):
    """optim.py:137-142: returns (lambdas, next_iteration)."""
    lr = scheduled_lr(hp, iteration, max_iters, iters_per_epoch)
    lambdas = apply_update(groups, hp, lr, iteration=iteration)
    return lambdas, iteration + 1


def tree_reduce(items, combine):
    """reduction.py:30-47: pairwise-left tree, odd trailing item carried."""
    items = list(items)
    if not items:
        raise ValueError("tree_reduce of empty list")
    while len(items) > 1:
        nxt = [combine(items[i], items[i + 1]) for i in range(0, len(items) - 1, 2)]
        if len(items) % 2:
            nxt.append(items[-1])
        items = nxt
    return items[0]


def all_reduce(grad_sets):
    """cluster.py:124-137: validate group names/shapes, then sum over workers."""
    ref = grad_sets[0]
    for j, g in enumerate(grad_sets[1:], start=1):
        if set(g) != set(ref):
            raise ValueError(f"worker {j} gradient groups differ from worker 0")
        for name in ref:
            if g[name].shape != ref[name].shape:
                raise ValueError(f"shape mismatch in group {name!r} on worker {j}")
    return tree_reduce(list(grad_sets), lambda a, b: {k: a[k] + b[k] for k in a})


def dp_step(replicas, grad_sets, hp, iteration, max_iters, iters_per_epoch, global_batch):
    """cluster.py:146-154: all_reduce -> / B -> lr -> identical update on every
    replica.  `replicas` is a list of group lists (one per worker)."""
    summed = all_reduce(grad_sets)                               # :146
    mean = {k: v / global_batch for k, v in summed.items()}      # :147-148
    lr = scheduled_lr(hp, iteration, max_iters, iters_per_epoch)  # :149
    lambdas = None
    for groups in replicas:                                      # :151
        for g in groups:                                         # nn.py:98-101
            np.copyto(g.grad, mean[g.name])
        lambdas = apply_update(groups, hp, lr, iteration=iteration)  # :153
    return lambdas, iteration + 1                                # :154


# ---------------------------------------------------------------------------
# Multi-threaded port (same arithmetic, groups split into element blocks) used
# only as the timed CPU baseline: the reference is single-threaded numpy, this
# gives it every host core.  Per-group norms are reduced from per-block fp64
# partial dot products, the update is elementwise per block.
# ---------------------------------------------------------------------------

def _blocks(n, block):
    return [(s, min(s + block, n)) for s in range(0, n, block)]


class ThreadedPort:
    def __init__(self, groups, threads, block=1 << 18):
        self.groups = groups
        self.threads = max(1, int(threads))
        self.pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None
        self.tasks = []
        for gi, g in enumerate(groups):
            for s, e in _blocks(g.param.size, block):
                self.tasks.append((gi, s, e))

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()

    def _map(self, fn, items):
        if self.pool is None:
            return [fn(t) for t in items]
        return list(self.pool.map(fn, items))

    def apply_update(self, hp, lr):
        groups = self.groups

        def norms(t):
            gi, s, e = t
            g = groups[gi]
            w = g.param.reshape(-1)[s:e]
            d = g.grad.reshape(-1)[s:e]
            return gi, float(w.dot(w)), float(d.dot(d))

        wsq = [0.0] * len(groups)
        gsq = [0.0] * len(groups)
        need = [hp.lars_enabled and g.category not in hp.lars_skip_categories for g in groups]
        for gi, a, b in self._map(norms, [t for t in self.tasks if need[t[0]]]):
            wsq[gi] += a
            gsq[gi] += b
        lams = [lars_from_sumsq(wsq[i], gsq[i], hp.weight_decay, hp.lars_trust) if need[i] else 1.0
                for i in range(len(groups))]

        def update(t):
            gi, s, e = t
            g = groups[gi]
            w = g.param.reshape(-1)[s:e]
            d = g.grad.reshape(-1)[s:e]
            m = g.momentum_buf.reshape(-1)[s:e]
            step_g = d + hp.weight_decay * w
            m *= hp.momentum
            m += (lams[gi] * lr) * step_g
            w -= m
            return bool(np.all(np.isfinite(w)))

        ok = self._map(update, self.tasks)
        return {g.name: lams[i] for i, g in enumerate(groups)}, all(ok)
