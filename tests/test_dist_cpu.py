"""Sharded data-parallel step on CPU: world_size 2 and 4 over gloo.

The CUDA kernels are replaced by a numpy stand-in (tests only) so the host
logic of cluster.DataParallelLars is checked without a GPU: shard layout,
segment clipping at shard edges, reduce-scatter of the summed gradient,
all-reduce of per-layer partial sums of squares, 1/B scaling, all-gather of
the updated shards.  The result must equal the oracle's replicated step
(cluster.py:146-153: all_reduce -> / B -> apply_update on every replica).
"""


import numpy as np
import pytest
import torch
import torch.distributed as dist

import gen
from helpers import HP, LAYOUTS, init_group, oracle_groups, spawn_ranks
from oracle import lars_oracle as orc


class NumpyKernels:
    """Test double for cluster.NativeKernels (same inputs and outputs)."""

    def __init__(self, hp, lr):
        self.hp, self.lr = hp, lr

    def partial_norms(self, eng, plan, ws, w_shard, g_shard, h):
        segs = eng.params.segments()
        sums = np.zeros((len(eng.params), 2))
        w = w_shard.numpy().astype(np.float64)
        g = g_shard.numpy().astype(np.float64)
        for off, ln, layer, _ in segs:
            sums[layer, 0] += float(w[off:off + ln] @ w[off:off + ln])
            sums[layer, 1] += float(g[off:off + ln] @ g[off:off + ln])
        eng.d_sumsq.copy_(torch.from_numpy(sums.reshape(-1)))

    def update(self, eng, plan, ws, w_shard, g_shard, m_shard, h):
        sums = eng.d_sumsq.numpy().reshape(-1, 2)
        lam = []
        for grp in eng.params:
            if not self.hp.lars_enabled or grp.category in self.hp.lars_skip_categories:
                lam.append(1.0)
            else:
                lam.append(orc.lars_from_sumsq(sums[grp.index, 0], sums[grp.index, 1] * h.grad_scale ** 2,
                                               self.hp.weight_decay, self.hp.lars_trust))
        eng.d_lambda.copy_(torch.tensor(lam, dtype=torch.float64))
        w = w_shard.numpy()
        g = g_shard.numpy()
        m = m_shard.numpy()
        for off, ln, layer, _ in eng.params.segments():
            sl = slice(off, off + ln)
            s = g[sl].astype(np.float64) * h.grad_scale + self.hp.weight_decay * w[sl]
            mn = self.hp.momentum * m[sl] + (lam[layer] * self.lr) * s
            m[sl] = mn
            w[sl] = w[sl] - mn


def _worker(rank, world, port, out_q, layout_name, seed):
    init_group("gloo", rank, world, port, out_q)
    from paper_1709_05011_b200 import cluster, optim
    from paper_1709_05011_b200.flat import FlatParamSet
    layout = LAYOUTS[layout_name]
    hp_kw = dict(base_lr=0.32, epochs=10, batch_size=512, warmup_epochs=2, lars_enabled=True)
    hp = optim.HyperParams(**hp_kw)
    st = optim.ScheduleState(100, 10, 7)
    fps = FlatParamSet(layout, "cpu", world_size=world, rank=rank)
    ins = gen.group_inputs(layout, seed)
    for grp, (w, _, m) in zip(fps, ins):
        grp.param.copy_(torch.from_numpy(w))
        fps.set_momentum(grp.name, m)
    # this rank's local (sum-convention) gradient
    for grp, g in zip(fps, gen.step_grads(layout, seed * 31 + rank, 0, g_scale=0.128)):
        grp.grad.copy_(torch.from_numpy(g))
    lr = optim.scheduled_lr(hp, st)
    B = 256 * world
    # the engine's device plan is not needed by the stand-in kernels
    from paper_1709_05011_b200 import flat as flatmod
    flatmod.LarsEngine.plan = lambda self, skip: (None, None)
    dp = cluster.DataParallelLars(fps, kernels=NumpyKernels(hp, lr))
    lams = dp.step(hp, st, grad_scale=1.0 / B)
    cluster.check_synchronized(fps)
    out_q.put((rank, fps.flat_param.numpy().copy(), fps.momentum.numpy().copy(),
               dict(lams), st.iteration, fps.shard_lo, fps.shard_hi))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,layout_name", [(2, "ragged"), (2, "mlp"), (4, "ragged"),
                                               (4, "mlp"), (8, "ragged"), (8, "mlp")])
def test_sharded_step_matches_replicated_oracle(layout_name, world):
    seed = 5
    res = spawn_ranks(_worker, world, (layout_name, seed), timeout=300)
    # oracle: replicated reference step on fp64 upcasts
    layout = LAYOUTS[layout_name]
    hp = HP(base_lr=0.32, epochs=10, batch_size=512, warmup_epochs=2, lars_enabled=True)
    groups = oracle_groups(layout, seed)
    sets = [{grp.name: g.astype(np.float64) for grp, g in
             zip(groups, gen.step_grads(layout, seed * 31 + r, 0, g_scale=0.128))} for r in range(world)]
    lam_ref, it = orc.dp_step([groups], sets, hp, 7, 100, 10, 256 * world)
    w_ref = np.concatenate([g.param.reshape(-1) for g in groups])
    m_ref = np.concatenate([g.momentum_buf.reshape(-1) for g in groups])
    # every rank holds identical full weights
    for r in range(1, world):
        assert np.array_equal(res[r][1], res[0][1])
    from paper_1709_05011_b200.flat import FlatParamSet
    fps = FlatParamSet(layout, "cpu")
    w_got = np.concatenate([res[0][1][g.offset:g.offset + g.numel] for g in fps])
    np.testing.assert_allclose(w_got, w_ref, rtol=1e-5, atol=1e-8)
    # momentum is sharded: stitch the shards back together
    m_full = np.zeros(max(res[r][6] for r in range(world)), dtype=np.float32)
    for r in range(world):
        lo, hi = res[r][5], res[r][6]
        m_full[lo:hi] = res[r][2]
    m_got = np.concatenate([m_full[g.offset:g.offset + g.numel] for g in fps])
    np.testing.assert_allclose(m_got, m_ref, rtol=1e-5, atol=1e-9)
    for k, v in lam_ref.items():
        assert res[0][3][k] == pytest.approx(v, rel=1e-6)  # fp32 gradient sum vs fp64
        for r in range(1, world):
            assert res[r][3][k] == res[0][3][k]
    assert res[0][4] == it == 8


def test_shard_segments_cover_every_element():
    from paper_1709_05011_b200 import layouts
    from paper_1709_05011_b200.flat import FlatParamSet
    layout = layouts.resnet50()
    for world in (1, 2, 4, 8):
        covered = np.zeros(FlatParamSet(layout, "cpu").padded_numel + 32 * 8, dtype=np.int32)
        for r in range(world):
            fps = FlatParamSet(layout, "cpu", world_size=world, rank=r)
            assert fps.shard_numel * world == fps.padded_numel
            assert fps.shard_lo % 32 == 0
            for off, ln, layer, _ in fps.segments():
                assert off % 4 == 0 and ln % 4 == 0
                covered[fps.shard_lo + off:fps.shard_lo + off + ln] += 1
        for g in FlatParamSet(layout, "cpu"):
            assert np.all(covered[g.offset:g.offset + g.numel] == 1), (world, g.name)


def _error_worker(rank, world, port, out_q):
    """Error paths of the product API across ranks (gloo): a replica whose
    weights drifted -> ConsistencyError naming it on every rank
    (cluster.py:101-107, reference pkg/tests/test_cluster.py:84-89); a
    FlatParamSet built for another world -> ProtocolError."""
    init_group("gloo", rank, world, port, out_q)
    from paper_1709_05011_b200 import cluster
    from paper_1709_05011_b200.errors import ConsistencyError, ProtocolError
    from paper_1709_05011_b200.flat import FlatParamSet
    layout = LAYOUTS["mlp"]
    fps = FlatParamSet(layout, "cpu", world_size=world, rank=rank)
    for grp, (w, _, _) in zip(fps, gen.group_inputs(layout, 3)):
        grp.param.copy_(torch.from_numpy(w))
    out = {}
    cluster.check_synchronized(fps)                  # identical replicas: no error
    out["sync_ok"] = True
    if rank == world - 1:                            # one element of the last rank drifts
        fps["dense3.weight"].param.view(-1)[17] += 1e-6
    try:
        cluster.check_synchronized(fps)
        out["desync"] = None
    except ConsistencyError as e:
        out["desync"] = str(e)
    wrong = FlatParamSet(layout, "cpu", world_size=world + 1, rank=rank)
    try:
        cluster.DataParallelLars(wrong)
        out["world_mismatch"] = None
    except ProtocolError as e:
        out["world_mismatch"] = str(e)
    other = FlatParamSet(layout, "cpu", world_size=world, rank=(rank + 1) % world)
    try:
        cluster.DataParallelLars(other)
        out["rank_mismatch"] = None
    except ProtocolError as e:
        out["rank_mismatch"] = str(e)
    out_q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_desync_and_group_mismatch_raise(world):
    res = {r: m[1] for r, m in spawn_ranks(_error_worker, world, (), timeout=300).items()}
    for r in range(world):
        assert res[r]["sync_ok"]
        # every rank raises, and the message names the drifted rank
        assert res[r]["desync"] is not None and str(world - 1) in res[r]["desync"], res[r]
        assert res[r]["world_mismatch"] is not None
        assert res[r]["rank_mismatch"] is not None
