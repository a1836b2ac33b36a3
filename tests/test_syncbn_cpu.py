"""Global-batch batch norm (syncbn.GlobalBatchNorm) against the
reference engine's own outputs: `nn.forward_backward_shards`
(pkg/src/batchlab/nn.py:250-367) run on 2 and 4 batch shards of a
dense -> batchnorm -> relu -> dense -> softmax-xent network
(tests/golden/make_bn_golden.py; vectors in syncbn_golden.npz).  Each
gloo rank (fp64, CPU) runs its shard through a torch model holding the same
weights; its local sum-convention gradients, the global loss and the BN
running statistics must match the reference's per-shard values."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from helpers import init_group, spawn_ranks

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "syncbn_golden.npz")


def _model(gold, group=None):
    from paper_1709_05011_b200.syncbn import GlobalBatchNorm
    nn = torch.nn
    m = nn.Sequential(nn.Linear(6, 5), GlobalBatchNorm(5, group=group), nn.ReLU(), nn.Linear(5, 3))
    m = m.double()
    with torch.no_grad():  # reference dense weights are (in, out)
        m[0].weight.copy_(torch.from_numpy(gold["init/dense0.weight"].T))
        m[0].bias.copy_(torch.from_numpy(gold["init/dense0.bias"]))
        m[1].weight.copy_(torch.from_numpy(gold["init/bn1.scale"]))
        m[1].bias.copy_(torch.from_numpy(gold["init/bn1.shift"]))
        m[3].weight.copy_(torch.from_numpy(gold["init/dense3.weight"].T))
        m[3].bias.copy_(torch.from_numpy(gold["init/dense3.bias"]))
    return m


def _grads(m):
    return {"dense0.weight": m[0].weight.grad.T.numpy(), "dense0.bias": m[0].bias.grad.numpy(),
            "bn1.scale": m[1].weight.grad.numpy(), "bn1.shift": m[1].bias.grad.numpy(),
            "dense3.weight": m[3].weight.grad.T.numpy(), "dense3.bias": m[3].bias.grad.numpy()}


def _worker(rank, world, port, q):
    init_group("gloo", rank, world, port, q)
    gold = dict(np.load(GOLD))
    m = _model(gold)
    x = torch.from_numpy(np.split(gold["x"], world)[rank])
    y = torch.from_numpy(np.split(gold["y"], world)[rank])
    loss = torch.nn.functional.cross_entropy(m(x), y, reduction="sum")
    loss.backward()
    total = loss.detach().clone()
    dist.all_reduce(total)
    q.put((rank, _grads(m), float(total), m[1].running_mean.numpy().copy(),
           m[1].running_var.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_global_bn_matches_reference_shards(world):
    gold = dict(np.load(GOLD))
    res = spawn_ranks(_worker, world, (), timeout=300)
    for r in range(world):
        _, grads, loss, rmean, rvar = res[r]
        for k, v in grads.items():
            np.testing.assert_allclose(v, gold[f"s{world}/grad{r}/{k}"], rtol=1e-10, atol=1e-13,
                                       err_msg=f"rank {r} {k}")
        assert loss == pytest.approx(float(gold[f"s{world}/loss"]), rel=1e-12)
        # running statistics from the global batch, biased variance, decay 0.9
        np.testing.assert_allclose(rmean, gold[f"s{world}/run_mean"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(rvar, gold[f"s{world}/run_var"], rtol=1e-12, atol=1e-15)


def test_single_process_global_bn_is_whole_batch():
    """World 1: the whole batch on one process == the sum of the reference's
    shard gradients (its shard layout does not change the math)."""
    gold = dict(np.load(GOLD))
    m = _model(gold)
    loss = torch.nn.functional.cross_entropy(m(torch.from_numpy(gold["x"])),
                                             torch.from_numpy(gold["y"]), reduction="sum")
    loss.backward()
    for k, v in _grads(m).items():
        ref = sum(gold[f"s2/grad{j}/{k}"] for j in range(2))
        np.testing.assert_allclose(v, ref, rtol=1e-10, atol=1e-13, err_msg=k)
    # eval mode uses the running statistics (nn.py predict_logits)
    m.eval()
    x = torch.from_numpy(gold["x"][:3])
    h = x @ m[0].weight.T + m[0].bias
    xhat = (h - m[1].running_mean) / torch.sqrt(m[1].running_var + 1e-5)
    ref = m[3](torch.relu(m[1].weight * xhat + m[1].bias))
    torch.testing.assert_close(m(x), ref)


def test_convert_global_bn_keeps_parameters_and_categories():
    from paper_1709_05011_b200.flat import FlatParamSet
    from paper_1709_05011_b200.syncbn import GlobalBatchNorm, convert_global_bn
    nn = torch.nn
    torch.manual_seed(0)
    m = nn.Sequential(nn.Conv2d(3, 4, 3), nn.BatchNorm2d(4), nn.ReLU(), nn.Flatten(), nn.Linear(4, 2))
    with torch.no_grad():
        m[1].weight.uniform_()
        m[1].running_mean.uniform_()
    w, rm = m[1].weight.clone(), m[1].running_mean.clone()
    m = convert_global_bn(m)
    assert isinstance(m[1], GlobalBatchNorm)
    assert torch.equal(m[1].weight, w) and torch.equal(m[1].running_mean, rm)
    cats = {g.name: g.category for g in FlatParamSet.from_module(m, "cpu")}
    assert cats["1.weight"] == "norm-scale" and cats["1.bias"] == "norm-shift"
    out = m(torch.randn(2, 3, 3, 3))
    assert out.shape == (2, 2)
