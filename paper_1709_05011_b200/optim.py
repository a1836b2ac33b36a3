"""Large-batch optimizer recipe with the LARS step on the B200.

Same public surface as the reference `batchlab.optim` (pkg/src/batchlab/
optim.py): `HyperParams`, `ScheduleState`, `linear_scaled_lr`,
`scheduled_lr`, `lars_local_lr`, `group_local_lr`, `apply_update`,
`sgd_step`, `max_iterations`, `schedule_table`, with the same validation and
errors.  The update itself runs as ONE fused sm_100a kernel launch over a
`FlatParamSet` (`liblars_b200.so`, include/lars_b200.h):

    lambda = trust * ||w|| / (||g|| + weight_decay * ||w||)   (fp64, per group)
    m <- momentum * m + lambda * lr * (g + weight_decay * w)   (fp32 state)
    w <- w - m

`sgd_step` evaluates the warmup + poly learning rate on the device from a
device iteration counter; the host only checks for schedule exhaustion
(`ScheduleExhaustedError`, raised before anything is launched, as in the
reference).  The returned lambdas are a lazily materialised mapping
name -> float.  Passing a reference `nn.ParamSet` of fp64 numpy arrays also
works (hostset.py): the caller's arrays are DMA'd to the device (pinned in
place), stepped, and written back in place.
"""

import math
import struct
from collections import OrderedDict
from collections.abc import Mapping
from dataclasses import dataclass

import torch

from . import _native as nat
from . import hostset
from .errors import ConfigError, DivergenceError, ScheduleExhaustedError
from .flat import FlatParamSet, _Plan, _ptr, _stream
from .layouts import BIAS, NORM_SCALE, NORM_SHIFT, WEIGHT

DEFAULT_LARS_SKIP = frozenset({BIAS, NORM_SCALE, NORM_SHIFT})  # optim.py:22


@dataclass
class HyperParams:
    """optim.py:25-55 (same fields, defaults and validation)."""

    base_lr: float
    epochs: int
    batch_size: int
    momentum: float = 0.9
    weight_decay: float = 0.0005
    poly_power: float = 2.0
    warmup_epochs: int = 0
    lars_enabled: bool = False
    lars_trust: float = 0.001
    lars_skip_categories: frozenset = DEFAULT_LARS_SKIP

    def __post_init__(self):
        if self.base_lr <= 0:
            raise ConfigError("base_lr must be positive")
        if not 0 <= self.momentum < 1:
            raise ConfigError("momentum must be in [0, 1)")
        if self.weight_decay < 0:
            raise ConfigError("weight_decay must be non-negative")
        if self.poly_power <= 0:
            raise ConfigError("poly_power must be positive")
        if self.epochs <= 0 or self.batch_size <= 0:
            raise ConfigError("epochs and batch_size must be positive")
        if not 0 <= self.warmup_epochs < self.epochs:
            raise ConfigError("need 0 <= warmup_epochs < epochs")
        if self.lars_trust <= 0:
            raise ConfigError("lars_trust must be positive")
        for v in (self.base_lr, self.momentum, self.weight_decay, self.poly_power, self.lars_trust):
            if not math.isfinite(v):
                raise ConfigError("hyperparameters must be finite")


@dataclass
class ScheduleState:
    """optim.py:58-66."""

    max_iterations: int
    iterations_per_epoch: int
    iteration: int = 0

    def __post_init__(self):
        if self.max_iterations <= 0 or self.iterations_per_epoch <= 0:
            raise ConfigError("schedule sizes must be positive")


def linear_scaled_lr(base_lr, base_batch, new_batch):
    """optim.py:69-73: batch k times bigger -> learning rate k times bigger."""
    if base_batch <= 0 or new_batch <= 0:
        raise ConfigError("batch sizes must be positive")
    return base_lr * (new_batch / base_batch)


def scheduled_lr(hp, st):
    """optim.py:76-95 on the host (the step evaluates the same expression on
    the device, `device_lr` in lars_kernels.cu)."""
    it = st.iteration
    if it > st.max_iterations:
        raise ScheduleExhaustedError(f"iteration {it} past schedule end {st.max_iterations}")
    warmup_iters = hp.warmup_epochs * st.iterations_per_epoch
    if it < warmup_iters:
        return hp.base_lr * (it + 1) / warmup_iters
    span = st.max_iterations - warmup_iters
    if span <= 0:
        return 0.0
    progress = (it - warmup_iters) / span
    return hp.base_lr * (1.0 - progress) ** hp.poly_power


def max_iterations(epochs, n, batch_size):
    """optim.py:145-147: floor(E * n / B)."""
    return (epochs * n) // batch_size


def schedule_table(hp, st_template):
    """optim.py:150-156: (iteration, lr) rows for the full schedule."""
    rows = []
    for it in range(st_template.max_iterations):
        st = ScheduleState(st_template.max_iterations, st_template.iterations_per_epoch, it)
        rows.append((it, scheduled_lr(hp, st)))
    return rows


def native_hparams(hp, st=None, *, lr=None, grad_scale=1.0, flags=0):
    """Pack HyperParams (+ schedule sizes) into the C struct lars_hparams_t."""
    h = nat.HParams()
    h.base_lr = float(hp.base_lr)
    h.momentum = float(hp.momentum)
    h.weight_decay = float(hp.weight_decay)
    h.poly_power = float(hp.poly_power)
    h.trust = float(hp.lars_trust)
    h.grad_scale = float(grad_scale)
    h.lr = float(lr) if lr is not None else 0.0
    if st is not None:
        h.warmup_iters = int(hp.warmup_epochs) * int(st.iterations_per_epoch)
        h.max_iters = int(st.max_iterations)
    h.lars_enabled = 1 if hp.lars_enabled else 0
    h.flags = flags | (nat.LARS_STEP_EXPLICIT_LR if lr is not None else 0)
    return h


def lambda_from_sums(w_sumsq, g_sumsq, weight_decay, trust, grad_scale=1.0):
    """optim.py:98-108 on reduced sums of squares (same roundings as the
    kernel's device_lambda)."""
    w_norm = math.sqrt(w_sumsq)
    g_norm = math.sqrt(g_sumsq) * abs(grad_scale)
    denom = g_norm + weight_decay * w_norm
    if w_norm == 0.0:
        return 0.0
    if denom == 0.0:
        return 1.0
    return trust * w_norm / denom


class LambdaMap(Mapping):
    """name -> lambda of one step, copied off the device on first access."""

    def __init__(self, names, dev_values):
        self._names = list(names)
        self._index = {n: i for i, n in enumerate(self._names)}
        self._dev = dev_values
        self._host = None

    def _values(self):
        if self._host is None:
            self._host = self._dev.cpu().tolist()
            self._dev = None
        return self._host

    def __getitem__(self, name):
        return self._values()[self._index[name]]

    def __iter__(self):
        return iter(self._names)

    def __len__(self):
        return len(self._names)

    def __repr__(self):
        return f"LambdaMap({dict(self)!r})"


# ---------------------------------------------------------------------------
# per-group trust ratio (lars_local_lr / group_local_lr)
# ---------------------------------------------------------------------------

_norm_plans = OrderedDict()  # (padded size, device) -> (plan, workspace), LRU
_NORM_PLANS_MAX = 8


def _sums_of_squares(param, grad):
    """Sum w^2 and Sum g^2 (fp64) of one tensor pair with the norm kernel."""
    dev = param.device if isinstance(param, torch.Tensor) and param.is_cuda else torch.device("cuda")
    w = torch.as_tensor(param).detach().reshape(-1).to(device=dev, dtype=torch.float32)
    g = torch.as_tensor(grad).detach().reshape(-1).to(device=dev, dtype=torch.float32)
    n = w.numel()
    npad = 1 << max(2, (n - 1).bit_length())  # power-of-two buckets (zero-padded)
    key = (npad, dev)
    if key not in _norm_plans:
        plan = _Plan([(0, npad, 0, WEIGHT)], 1, frozenset())
        ws = torch.empty(int(plan.info.workspace_bytes), dtype=torch.uint8, device=dev)
        nat.check(nat.load().lars_workspace_init(plan.handle, _ptr(ws), _stream()))
        _norm_plans[key] = (plan, ws)
        while len(_norm_plans) > _NORM_PLANS_MAX:
            _norm_plans.popitem(last=False)
    _norm_plans.move_to_end(key)
    plan, ws = _norm_plans[key]
    buf = torch.zeros(2, npad, dtype=torch.float32, device=dev)
    buf[0, :n] = w
    buf[1, :n] = g
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    it = torch.zeros(1, dtype=torch.int64, device=dev)
    info = torch.zeros(nat.STEP_INFO_BYTES, dtype=torch.uint8, device=dev)
    h = nat.HParams()
    h.flags = nat.LARS_STEP_EXPLICIT_LR
    nat.check(nat.load().lars_partial_norms(plan.handle, _ptr(buf[0]), _ptr(buf[1]),
                                            nat.ctypes.byref(h), _ptr(it), _ptr(sums),
                                            _ptr(info), _ptr(ws), _stream()))
    s = sums.cpu().tolist()
    return s[0], s[1]


def lars_local_lr(param, grad, weight_decay, trust):
    """optim.py:98-108: layer-wise trust ratio for one parameter group."""
    w2, g2 = _sums_of_squares(param, grad)
    return lambda_from_sums(w2, g2, weight_decay, trust)


def group_local_lr(group, hp):
    """optim.py:111-114."""
    if not hp.lars_enabled or group.category in hp.lars_skip_categories:
        return 1.0
    return lars_local_lr(group.param, group.grad, hp.weight_decay, hp.lars_trust)


# ---------------------------------------------------------------------------
# the step
# ---------------------------------------------------------------------------

def _launch_fused(params, hp, st, *, lr, grad_scale, advance):
    """Queue one lars_step launch on the current stream; returns the engine."""
    if params.world_size != 1:
        raise ConfigError("a sharded FlatParamSet steps through cluster.DataParallelLars")
    eng = params.engine()
    key = frozenset(hp.lars_skip_categories)
    plan, ws = eng.plan(key)
    flags = nat.LARS_STEP_ADVANCE_ITER if advance else 0
    if eng.carry_valid(key):
        flags |= nat.LARS_STEP_USE_WCARRY
    h = native_hparams(hp, st, lr=lr, grad_scale=grad_scale, flags=flags)
    nat.check(nat.load().lars_step(
        plan.handle, _ptr(params.flat_param), _ptr(params.flat_grad), _ptr(params.momentum),
        nat.ctypes.byref(h), _ptr(eng.d_iter), _ptr(eng.d_sumsq), _ptr(eng.d_lambda),
        _ptr(eng.d_info), _ptr(ws), _stream()))
    eng.mark_carry(key)
    return eng


def apply_update(params, hp, lr, iteration=0, *, grad_scale=1.0, check=True):
    """optim.py:117-134: one momentum step at the given learning rate;
    returns the per-group lambdas.

    `params` is a FlatParamSet (device-resident, the fast path) or any
    reference-style ParamSet of numpy arrays (copied in and back out).
    `grad_scale` multiplies the gradient (1/B for a summed gradient).  With
    `check=True` a non-finite update raises DivergenceError(iteration) like
    the reference (this reads one small status word back); with
    `check=False` call `check_divergence(params, iteration)` later.
    """
    if not isinstance(params, FlatParamSet):
        # reference-style ParamSet of caller-owned fp64 arrays (hostset.py):
        # DMA in, one step, then write back the groups the reference would
        # have updated -- all of them, or up to the first non-finite one
        # (optim.py:125-133) -- and raise as it does
        mirror, groups = hostset.mirror_for(params)

        def launch(fps):
            return _launch_fused(fps, hp, None, lr=lr, grad_scale=grad_scale, advance=False)

        out, bad = mirror.step(groups, hp, lr, iteration, grad_scale, check, launch)
        if check and bad is not None:
            raise DivergenceError(iteration, f"group {mirror.names[bad]} non-finite at iteration "
                                             f"{iteration}")
        return out
    eng = _launch_fused(params, hp, None, lr=lr, grad_scale=grad_scale, advance=False)
    lams = LambdaMap(params.names(), eng.d_lambda.clone())
    if check:
        eng.raise_if_diverged(iteration)
    return lams


def sgd_step(params, hp, st, *, grad_scale=1.0, check=True):
    """optim.py:137-142: scheduled momentum/LARS step; advances st.iteration.

    The lr is evaluated on the device from the device iteration counter; the
    host raises ScheduleExhaustedError before launching if the schedule is
    exhausted, and (with check=True) DivergenceError without advancing
    st.iteration, as the reference does."""
    scheduled_lr(hp, st)  # host-side exhaustion check (optim.py:84-87)
    if not isinstance(params, FlatParamSet):
        lams = apply_update(params, hp, scheduled_lr(hp, st), iteration=st.iteration,
                            grad_scale=grad_scale, check=check)
        st.iteration += 1
        return lams
    eng = params.engine()
    eng.set_iteration(st.iteration)
    _launch_fused(params, hp, st, lr=None, grad_scale=grad_scale, advance=True)
    eng.host_iter = st.iteration + 1
    lams = LambdaMap(params.names(), eng.d_lambda.clone())
    if check:
        eng.raise_if_diverged(st.iteration)
    st.iteration += 1
    return lams


def check_divergence(params, iteration):
    """Raise DivergenceError(iteration) if the last step produced non-finite
    weights (deferred form of the check at optim.py:132-133)."""
    if not isinstance(params, FlatParamSet):
        mirror = hostset.mirror_of(params)
        if mirror is not None and mirror.last_bad is not None:
            raise DivergenceError(iteration, f"group {mirror.names[mirror.last_bad]} non-finite "
                                             f"at iteration {iteration}")
        return
    params.engine().raise_if_diverged(iteration)


def step_info(params):
    """(lr, iteration, nonfinite_layer, status) of the last step (blocking)."""
    return params.engine().read_info()
