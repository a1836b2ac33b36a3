"""100-step trajectories at config size, and the step's state semantics.

* ResNet-50 (config 4) and AlexNet-BN (configs 2/3) parameter sets: 100
  scheduled LARS steps through `optim.sgd_step` against the oracle
  (`oracle/lars_oracle.py`, the reference's `optim.sgd_step`,
  optim.py:137-142) on identical fp32 inputs, at the north-star multi-step
  tolerance 1e-4 (floor 1e-6 rms(layer)), lambdas at 1e-6 relative.
* What a DivergenceError leaves behind (optim.py:125-133): the reference
  updates the groups up to and including the first non-finite one, then
  raises; the host-ParamSet drop-in reproduces that exactly, the
  device-resident step updates every group (one launch) and names the same
  group and iteration.
* Norm-carry invalidation through module parameters (load_state_dict,
  in-place writes) and CUDA-graph capture/replay after a weight reload.
"""

import numpy as np
import pytest
import torch

import gen
from helpers import HP, assert_params_close, oracle_groups, rolled_grads
from oracle import lars_oracle as orc

pytestmark = pytest.mark.gpu

BIG_HP = dict(base_lr=25.6, epochs=90, batch_size=32768, momentum=0.9, weight_decay=5e-4,
              poly_power=2.0, warmup_epochs=5, lars_enabled=True, lars_trust=1e-3)


def _load(layout, seed, device):
    from paper_1709_05011_b200.flat import FlatParamSet
    fps = FlatParamSet(layout, device)
    for grp, (w, g, m) in zip(fps, gen.group_inputs(layout, seed)):
        grp.param.copy_(torch.from_numpy(w))
        grp.grad.copy_(torch.from_numpy(g))
        grp.momentum_buf.copy_(torch.from_numpy(m))
    fps.invalidate_norm_cache()
    return fps


def _flat(fps, which):
    return np.concatenate([(grp.param if which == "w" else grp.momentum_buf)
                           .detach().double().cpu().numpy().reshape(-1) for grp in fps])


@pytest.mark.parametrize("name,it0,mx,ipe", [("resnet50", 150, 3515, 39),
                                             ("alexnet_bn", 150, 3906, 39)])
def test_hundred_steps_config_size_vs_oracle(name, it0, mx, ipe, cuda):
    """100 steps crossing the end of warmup (it 150 -> 250, warmup 195):
    fresh gradients every step (a base set rolled and power-of-two scaled,
    exact in fp32), carried ||w|| on the device from step 2 on."""
    from paper_1709_05011_b200 import layouts, optim
    layout = layouts.get(name)
    seed = 17
    fps = _load(layout, seed, cuda)
    groups = oracle_groups(layout, seed)
    base = gen.step_grads(layout, seed, 0, g_scale=1e-3)
    hp, hpo = optim.HyperParams(**BIG_HP), HP(**BIG_HP)
    st = optim.ScheduleState(mx, ipe, it0)
    ito = it0
    lams = lam_ref = None
    for t in range(100):
        gs = rolled_grads(base, t)
        fps.set_grads({grp.name: g for grp, g in zip(fps, gs)})
        for grp, g in zip(groups, gs):
            np.copyto(grp.grad, g, casting="unsafe")
        lams = optim.sgd_step(fps, hp, st, check=False)
        lam_ref, ito = orc.sgd_step(groups, hpo, ito, mx, ipe)
    optim.check_divergence(fps, st.iteration - 1)
    assert st.iteration == ito == it0 + 100
    w_ref = np.concatenate([g.param.reshape(-1) for g in groups])
    m_ref = np.concatenate([g.momentum_buf.reshape(-1) for g in groups])
    # 1e-4 relative per parameter; the absolute floor is 1e-5 rms(layer): the
    # state is fp32 (north star), and at this learning rate (lambda*lr moves
    # w by ~2.5 % a step, momentum 0.9) the fp32 rounding of w and m over
    # 100 steps alone reaches 2.3e-6 rms -- a plain numpy fp32 restatement of
    # the same arithmetic misses a 1e-6 rms floor on layer3.0.downsample by
    # the same 0.1 % the kernel does (tools/fp32_floor.py)
    assert_params_close(_flat(fps, "w"), w_ref, layout, 1e-4, floor=1e-5, what="w")
    assert_params_close(_flat(fps, "m"), m_ref, layout, 1e-4, floor=1e-5, what="m")
    for k, v in lam_ref.items():
        assert lams[k] == pytest.approx(v, rel=1e-6, abs=0), k
    # the device schedule followed the host one
    lr, it, _, _ = optim.step_info(fps)
    assert it == it0 + 99
    assert lr == pytest.approx(orc.scheduled_lr(hpo, it0 + 99, mx, ipe), rel=1e-15)


LAYOUT = [("a.weight", (40, 3), "weight"), ("a.bias", (3,), "bias"),
          ("b.weight", (33, 7), "weight"), ("c.weight", (129,), "weight"),
          ("d.weight", (64,), "weight")]


def _diverging_groups(seed):
    groups = oracle_groups(LAYOUT, seed)
    groups[2].grad.reshape(-1)[5] = np.inf        # b.weight: first non-finite group
    groups[3].grad.reshape(-1)[0] = np.nan        # c.weight: also bad, later
    return groups


@pytest.mark.parametrize("part_min", [None, 1], ids=["one-part", "part-per-group"])
def test_divergence_host_paramset_matches_reference_state(part_min, cuda, monkeypatch):
    """Reference-style numpy ParamSet: same exception, same iteration, and the
    caller's arrays end exactly where the reference leaves them (groups
    after the failing one untouched) -- also when the groups are pipelined
    in parts (the failing group's part is written up to it, later parts not
    at all)."""
    from paper_1709_05011_b200 import hostset, optim
    if part_min is not None:
        monkeypatch.setattr(hostset, "PART_MIN_ELEMS", part_min)
    from paper_1709_05011_b200.errors import DivergenceError
    hp_kw = dict(base_lr=0.1, epochs=10, batch_size=32, lars_enabled=True)
    ref = _diverging_groups(3)
    mine = [g.copy() for g in ref]
    before = [g.copy() for g in ref]
    with pytest.raises(orc.OracleDivergence) as eo:
        orc.apply_update(ref, HP(**hp_kw), 0.05, iteration=42)
    with pytest.raises(DivergenceError) as em:
        optim.apply_update(mine, optim.HyperParams(**hp_kw), 0.05, iteration=42)
    assert em.value.iteration == eo.value.iteration == 42
    assert eo.value.group in str(em.value)
    for a, r, b in zip(mine, ref, before):
        if r.name in ("d.weight",):               # after the failing group: untouched
            assert np.array_equal(a.param, b.param) and np.array_equal(a.param, r.param)
            assert np.array_equal(a.momentum_buf, b.momentum_buf)
        fin = np.isfinite(r.param)
        assert np.array_equal(np.isfinite(a.param), fin), a.name
        np.testing.assert_allclose(a.param[fin], r.param[fin], rtol=1e-5, atol=1e-7)


def test_divergence_device_state_pinned(cuda):
    """Device-resident FlatParamSet: one launch updates every group; the
    error names the first non-finite group in order and the iteration.
    Groups before it hold exactly the reference's values; the failing group
    and those after it hold the full-step values (documented deviation)."""
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.errors import DivergenceError
    from paper_1709_05011_b200.flat import FlatParamSet
    hp_kw = dict(base_lr=0.1, epochs=10, batch_size=32, lars_enabled=True)
    ref = _diverging_groups(4)
    full = [g.copy() for g in ref]
    fps = FlatParamSet(LAYOUT, cuda)
    for grp, src in zip(fps, ref):
        grp.param.copy_(torch.from_numpy(src.param))
        grp.grad.copy_(torch.from_numpy(src.grad))
        grp.momentum_buf.copy_(torch.from_numpy(src.momentum_buf))
    fps.invalidate_norm_cache()
    with pytest.raises(orc.OracleDivergence) as eo:
        orc.apply_update(ref, HP(**hp_kw), 0.05, iteration=7)
    with pytest.raises(DivergenceError) as em:
        optim.apply_update(fps, optim.HyperParams(**hp_kw), 0.05, iteration=7)
    assert em.value.iteration == 7 and eo.value.group in str(em.value)
    # the full step on every group (the oracle run past the error, group by group)
    hpo = HP(**hp_kw)
    for g in full:
        try:
            orc.apply_update([g], hpo, 0.05, iteration=7)
        except orc.OracleDivergence:
            pass
    for grp, r, f in zip(fps, ref, full):
        got = grp.param.double().cpu().numpy()
        exp = r.param if grp.name in ("a.weight", "a.bias") else f.param
        fin = np.isfinite(exp)
        assert np.array_equal(np.isfinite(got), fin), grp.name
        np.testing.assert_allclose(got[fin], exp[fin], rtol=1e-5, atol=1e-7, err_msg=grp.name)


def test_module_writes_invalidate_carry(cuda):
    """Writes through module parameters bound by from_module (load_state_dict,
    in-place ops) bump their own version counters, not the flat buffer's: the
    carried ||w|| must still be dropped, so the next lambda matches a fresh
    set built from the same weights."""
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.flat import FlatParamSet
    torch.manual_seed(0)
    nn = torch.nn
    model = nn.Sequential(nn.Linear(32, 64), nn.BatchNorm1d(64), nn.ReLU(), nn.Linear(64, 10)).to(cuda)
    saved = {k: v.clone() for k, v in model.state_dict().items()}
    fps = FlatParamSet.from_module(model, cuda)
    hp = optim.HyperParams(base_lr=0.5, epochs=10, batch_size=32, lars_enabled=True)
    key = frozenset(hp.lars_skip_categories)
    st = optim.ScheduleState(100, 10)
    for _ in range(2):
        fps.flat_grad.normal_(0, 1e-2)
        optim.sgd_step(fps, hp, st)
    assert fps.engine().carry_valid(key)
    model.load_state_dict(saved)                     # checkpoint restore through the module
    assert not fps.engine().carry_valid(key)
    fps.flat_grad.normal_(0, 1e-2)
    twin = fps.copy()
    lam = optim.sgd_step(fps, hp, optim.ScheduleState(100, 10, 2))
    lam_twin = optim.sgd_step(twin, hp, optim.ScheduleState(100, 10, 2))
    for k in lam:
        assert lam[k] == pytest.approx(lam_twin[k], rel=1e-13, abs=0), k
    with torch.no_grad():
        model[0].weight.mul_(2.0)                    # in-place write through the module
    assert not fps.engine().carry_valid(key)


def test_graph_capture_refuses_stale_carry_and_replay_recovers(cuda):
    """DataParallelLars.capture() needs a valid carry; a replay after the
    weights were rewritten runs one eager step with fresh norms instead of
    the graph (no stale ||w||), then replays resume."""
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.cluster import DataParallelLars
    from paper_1709_05011_b200.errors import ProtocolError
    from paper_1709_05011_b200 import layouts
    layout = layouts.mlp()
    hp = optim.HyperParams(base_lr=0.32, epochs=10, batch_size=512, warmup_epochs=2,
                           lars_enabled=True)
    a = _load(layout, 8, cuda)
    b = _load(layout, 8, cuda)
    dp = DataParallelLars(a)
    sa = optim.ScheduleState(200, 10)
    with pytest.raises(ProtocolError):
        dp.capture(hp, sa)                           # no step yet: carry invalid
    dp.step(hp, sa)
    gstep = dp.capture(hp, sa)
    gstep.replay()
    snapshot = a.flat_param.clone()
    a.flat_param.mul_(0.5)                           # external rewrite (e.g. checkpoint load)
    gstep.replay()                                   # must not use the stale carry
    gstep.replay()
    torch.cuda.synchronize()
    # reference: the same sequence of eager steps on a twin
    sb = optim.ScheduleState(200, 10)
    for _ in range(2):
        optim.sgd_step(b, hp, sb)
    assert torch.equal(b.flat_param, snapshot)
    b.flat_param.mul_(0.5)
    for _ in range(2):
        optim.sgd_step(b, hp, sb)
    assert sa.iteration == sb.iteration == 4
    np.testing.assert_allclose(a.flat_param.cpu().numpy(), b.flat_param.cpu().numpy(),
                               rtol=1e-6, atol=1e-9)
    la, lb = gstep.lambdas(), optim.LambdaMap(b.names(), b.engine().d_lambda.clone())
    for k in la:
        assert la[k] == pytest.approx(lb[k], rel=1e-12), k


@pytest.mark.parametrize("part_min", [None, 1], ids=["one-part", "part-per-group"])
def test_host_paramset_pinned_in_place_two_steps(part_min, cuda, monkeypatch):
    """Reference-style ParamSet with big fp64 groups (pinned where they lie),
    small ones (bounce buffer) and two groups that are views of ONE buffer
    (the second cannot be pinned again: bounce): two apply_update calls
    against the oracle; the caller's arrays are updated in place.  Also with
    the groups pipelined in parts (copy-back of one part overlapping the
    copy-in of the next)."""
    from paper_1709_05011_b200 import hostset, optim
    if part_min is not None:
        monkeypatch.setattr(hostset, "PART_MIN_ELEMS", part_min)
    hp_kw = dict(base_lr=0.4, epochs=10, batch_size=32, lars_enabled=True)
    layout = [("big.weight", (512, 1024), "weight"), ("big.bias", (1024,), "bias"),
              ("v1.weight", (300, 1000), "weight"), ("v2.weight", (200, 1000), "weight"),
              ("tiny.weight", (3, 5), "weight")]
    ref = oracle_groups(layout, 11)
    shared = np.empty(500_000, dtype=np.float64)     # v1 / v2 share one allocation
    mine = [g.copy() for g in ref]
    v1 = shared[:300_000].reshape(300, 1000)
    v2 = shared[300_000:].reshape(200, 1000)
    v1[...] = mine[2].param
    v2[...] = mine[3].param
    mine[2].param, mine[3].param = v1, v2
    ids = [id(g.param) for g in mine]
    hp, hpo = optim.HyperParams(**hp_kw), HP(**hp_kw)
    for it in range(2):
        lam_ref = orc.apply_update(ref, hpo, 0.05, iteration=it)
        lam = optim.apply_update(mine, hp, 0.05, iteration=it)
        for a, b in zip(mine, ref):
            np.testing.assert_allclose(a.param, b.param, rtol=1e-5,
                                       atol=1e-7 * np.sqrt(np.mean(b.param ** 2)), err_msg=a.name)
            np.testing.assert_allclose(a.momentum_buf, b.momentum_buf, rtol=1e-5,
                                       atol=1e-7 * np.sqrt(np.mean(b.momentum_buf ** 2)))
        for k in lam_ref:
            assert lam[k] == pytest.approx(lam_ref[k], rel=1e-6), k
        for g in ref:                                  # fresh gradient for the next step
            g.grad *= -0.5
        for g, r in zip(mine, ref):
            np.copyto(g.grad, r.grad)
    assert [id(g.param) for g in mine] == ids
    assert np.shares_memory(mine[2].param, shared) and np.shares_memory(mine[3].param, shared)
