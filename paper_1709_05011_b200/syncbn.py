"""Global-batch batch normalisation across data-parallel ranks.

The reference normalises with statistics of the GLOBAL batch, every worker's
shard included (pkg/src/batchlab/nn.py:289-310 forward, :356-367 backward):

    s1 = sum x,  s2 = sum x^2            over all shards    (nn.py:294-295)
    mean = s1 / n,  var = max(s2/n - mean^2, 0)   (biased)  (:296-297)
    xhat = (x - mean) / sqrt(var + eps),  y = scale * xhat + shift
    running mean / var <- 0.9 * running + 0.1 * batch       (:309-310, BN_MOMENTUM = 0.9)
    backward (sum convention): T1 = sum dy, T2 = sum dy * xhat over all shards,
    dx = scale / sqrt(var + eps) * (dy - T1/n - xhat * T2/n); each shard's
    scale / shift gradient is its LOCAL sum (dy * xhat, dy)  (:356-367)

`GlobalBatchNorm` does exactly that with one all-reduce of [s1 | s2 | n] in
forward and one of [T1 | T2] in backward over the process group (torch's
SyncBatchNorm differs: unbiased running variance, momentum 0.1 of the new
value, and it averages rather than sums).  Statistics are per channel over
every other dimension, so it serves dense (N, C) and conv (N, C, H, W)
layers.  With micro-batch accumulation the "global batch" of one
normalisation is the P micro-batches processed together.
"""

import torch
import torch.distributed as dist

BN_MOMENTUM = 0.9  # nn.py:31 -- fraction of the running statistic kept
BN_EPS = 1e-5      # nn.py:30


def _all_reduce(t, group):
    if group is not False and dist.is_available() and dist.is_initialized() \
            and dist.get_world_size(group) > 1:
        dist.all_reduce(t, group=group)
    return t


class _GlobalBNFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, scale, shift, eps, group):
        c = x.shape[1]
        dims = [d for d in range(x.dim()) if d != 1]
        shape = [1, c] + [1] * (x.dim() - 2)
        n_local = x.numel() // c
        stats = torch.cat([x.sum(dims), (x * x).sum(dims),
                           torch.full((1,), float(n_local), dtype=x.dtype, device=x.device)])
        stats = _all_reduce(stats, group)
        n = stats[2 * c]
        mean = stats[:c] / n
        var = torch.clamp(stats[c:2 * c] / n - mean * mean, min=0.0)
        inv = 1.0 / torch.sqrt(var + eps)
        xhat = (x - mean.view(shape)) * inv.view(shape)
        ctx.save_for_backward(xhat, inv, scale)
        ctx.group, ctx.n, ctx.dims, ctx.shape = group, n, dims, shape
        ctx.mark_non_differentiable(mean, var)
        return scale.view(shape) * xhat + shift.view(shape), mean, var

    @staticmethod
    def backward(ctx, dy, _dmean, _dvar):
        xhat, inv, scale = ctx.saved_tensors
        dims, shape, n = ctx.dims, ctx.shape, ctx.n
        c = xhat.shape[1]
        t1 = dy.sum(dims)
        t2 = (dy * xhat).sum(dims)
        tot = _all_reduce(torch.cat([t1, t2]), ctx.group)
        big_t1, big_t2 = tot[:c], tot[c:]
        dx = (scale * inv).view(shape) * (dy - (big_t1 / n).view(shape) - xhat * (big_t2 / n).view(shape))
        return dx, t2, t1, None, None


class GlobalBatchNorm(torch.nn.modules.batchnorm._BatchNorm):
    """BatchNorm over the global batch of all ranks in `group` with the
    reference's semantics (biased variance, running decay 0.9).  A
    `torch.nn.modules.batchnorm._BatchNorm` so FlatParamSet files its weight /
    bias as norm-scale / norm-shift (the LARS skip set, optim.py:22)."""

    def __init__(self, num_features, eps=BN_EPS, group=None, device=None, dtype=None):
        super().__init__(num_features, eps=eps, momentum=1.0 - BN_MOMENTUM, affine=True,
                         track_running_stats=True, device=device, dtype=dtype)
        self.group = group

    def _check_input_dim(self, x):
        if x.dim() < 2:
            raise ValueError(f"expected at least 2-D input, got {x.dim()}-D")

    def forward(self, x):
        self._check_input_dim(x)
        shape = [1, x.shape[1]] + [1] * (x.dim() - 2)
        if not self.training:  # eval: running statistics (nn.py predict_logits)
            xhat = (x - self.running_mean.view(shape)) / torch.sqrt(self.running_var.view(shape) + self.eps)
            return self.weight.view(shape) * xhat + self.bias.view(shape)
        y, mean, var = _GlobalBNFn.apply(x, self.weight, self.bias, self.eps, self.group)
        with torch.no_grad():
            self.running_mean.mul_(BN_MOMENTUM).add_((1.0 - BN_MOMENTUM) * mean)
            self.running_var.mul_(BN_MOMENTUM).add_((1.0 - BN_MOMENTUM) * var)
            self.num_batches_tracked += 1
        return y


def convert_global_bn(module, group=None):
    """Replace every torch BatchNorm{1,2,3}d / SyncBatchNorm in `module` by a
    GlobalBatchNorm with the same parameters and running statistics."""
    bn_types = (torch.nn.BatchNorm1d, torch.nn.BatchNorm2d, torch.nn.BatchNorm3d,
                torch.nn.SyncBatchNorm)
    if isinstance(module, bn_types) and not isinstance(module, GlobalBatchNorm):
        out = GlobalBatchNorm(module.num_features, eps=module.eps, group=group,
                              device=module.weight.device if module.affine else None,
                              dtype=module.weight.dtype if module.affine else None)
        with torch.no_grad():
            if module.affine:
                out.weight.copy_(module.weight)
                out.bias.copy_(module.bias)
            if module.track_running_stats:
                out.running_mean.copy_(module.running_mean)
                out.running_var.copy_(module.running_var)
        out.train(module.training)
        return out
    for name, child in module.named_children():
        setattr(module, name, convert_global_bn(child, group))
    return module
