"""Pin the CPU oracle (oracle/lars_oracle.py) before trusting it.

1. The reference's own known-answer tests, restated on the oracle
   (pkg/tests/test_optim.py:17-222, test_cluster.py:93-105,
   test_acceptance.py:166-182).
2. Golden vectors produced by running the reference itself
   (tests/golden/make_golden.py): the oracle must reproduce them exactly
   (same fp64 operations in the same order).
"""

import numpy as np
import pytest

from helpers import HP, manifest, golden_arrays, run_oracle_case
from oracle import lars_oracle as orc


def hp(**kw):
    base = dict(base_lr=0.1, epochs=10, batch_size=32)
    base.update(kw)
    return HP(**base)


# ---- test_optim.py:16-36 linear scaling ----
def test_linear_scaling_kats():
    assert orc.linear_scaled_lr(0.02, 512, 4096) == 0.16
    assert orc.linear_scaled_lr(0.02, 512, 512) == 0.02
    assert orc.linear_scaled_lr(0.2, 256, 32768) == 25.6
    with pytest.raises(ValueError):
        orc.linear_scaled_lr(0.1, 0, 64)


# ---- test_optim.py:38-89 schedule ----
def test_schedule_kats():
    h = hp(base_lr=0.4, poly_power=2.0)
    assert orc.scheduled_lr(h, 0, 100, 10) == 0.4
    assert orc.scheduled_lr(h, 100, 100, 10) == 0.0
    assert orc.scheduled_lr(h, 50, 100, 10) == pytest.approx(0.1, rel=1e-12)
    h = hp(base_lr=0.8, warmup_epochs=2)
    assert orc.scheduled_lr(h, 0, 100, 10) == pytest.approx(0.8 / 20)
    assert orc.scheduled_lr(h, 19, 100, 10) == 0.8
    assert orc.scheduled_lr(h, 20, 100, 10) == 0.8
    lrs = [orc.scheduled_lr(h, it, 200, 10) for it in range(20, 201)]
    assert all(a >= b for a, b in zip(lrs, lrs[1:]))
    h = hp(base_lr=1.0, warmup_epochs=3)
    prev = None
    for it in range(61):
        lr = orc.scheduled_lr(h, it, 60, 5)
        if prev is not None:
            assert abs(lr - prev) <= 1.0 / 15 + 1e-12
        prev = lr
    with pytest.raises(orc.OracleScheduleExhausted):
        orc.scheduled_lr(hp(), 11, 10, 5)
    assert orc.max_iterations(50, 9000, 32) == 14062
    assert orc.max_iterations(1, 64, 64) == 1


def test_acceptance_c8_schedule_contract():
    h = hp(base_lr=0.4, poly_power=2.0, warmup_epochs=2)
    assert orc.scheduled_lr(h, 0, 100, 10) == pytest.approx(0.4 / 20)
    assert orc.scheduled_lr(h, 19, 100, 10) == 0.4
    assert orc.scheduled_lr(h, 20, 100, 10) == 0.4
    assert orc.scheduled_lr(h, 100, 100, 10) == 0.0


# ---- test_optim.py:99-131 LARS ----
def test_lars_kats():
    assert orc.lars_local_lr(np.array([1.0]), np.array([1.0]), 0.0, 0.001) == 0.001
    assert orc.lars_local_lr(np.zeros(4), np.ones(4), 0.0, 0.01) == 0.0
    assert orc.lars_local_lr(np.array([2.0]), np.array([1.0]), 0.5, 0.01) == pytest.approx(0.01, rel=1e-12)
    assert orc.lars_local_lr(np.array([3.0]), np.zeros(1), 0.0, 0.01) == 1.0
    w, g = np.array([3.0, 4.0]), np.array([1.0, 2.0])
    lam = orc.lars_local_lr(w, g, 0.0, 0.001)
    for c in (0.01, 1.7, 100.0):
        assert orc.lars_local_lr(c * w, c * g, 0.0, 0.001) == pytest.approx(lam, rel=1e-12)


def test_lars_from_sumsq_matches_norm_form():
    rng = np.random.default_rng(0)
    for _ in range(20):
        w, g = rng.standard_normal(100), rng.standard_normal(100) * 1e-3
        a = orc.lars_local_lr(w, g, 5e-4, 1e-3)
        b = orc.lars_from_sumsq(float(w @ w), float(g @ g), 5e-4, 1e-3)
        assert a == pytest.approx(b, rel=1e-14)


def test_skip_categories_unit_lambda():
    h = hp(lars_enabled=True)
    for cat in ("bias", "norm-scale", "norm-shift"):
        grp = orc.Group("x", np.ones(3), np.ones(3), np.zeros(3), cat)
        assert orc.group_local_lr(grp, h) == 1.0
    grp = orc.Group("x", np.ones(3), np.ones(3), np.zeros(3), "weight")
    assert orc.group_local_lr(grp, h) != 1.0


# ---- test_optim.py:134-214 update algebra ----
def _one(w, g):
    return [orc.Group("dense0.weight", np.array(w, float), np.array(g, float),
                      np.zeros(len(w)), "weight")]


def test_vanilla_step_subtracts_gradient():
    gs = _one([0.5, -1.0, 2.0], [0.25] * 3)
    before = gs[0].param.copy()
    orc.apply_update(gs, hp(base_lr=1.0, momentum=0.0, weight_decay=0.0), lr=1.0)
    assert np.array_equal(gs[0].param, before - 0.25)


def test_momentum_unrolled_two_steps():
    gs = _one([0.5, -1.0], [0.5, 0.5])
    before = gs[0].param.copy()
    h = hp(base_lr=0.1, momentum=0.9, weight_decay=0.0)
    for _ in range(2):
        gs[0].grad[:] = 0.5
        orc.apply_update(gs, h, lr=0.1)
    assert gs[0].param == pytest.approx(before - 0.1 * 0.5 * 2.9, rel=1e-12)


def test_lars_scales_update_magnitude():
    rng = np.random.default_rng(0)
    gs = _one(rng.uniform(-1, 1, 6), rng.standard_normal(6))
    w_norm, g_norm = np.linalg.norm(gs[0].param), np.linalg.norm(gs[0].grad)
    before, grad = gs[0].param.copy(), gs[0].grad.copy()
    orc.apply_update(gs, hp(momentum=0.0, weight_decay=0.0, lars_enabled=True, lars_trust=0.02), lr=0.1)
    assert before - gs[0].param == pytest.approx(0.02 * w_norm / g_norm * 0.1 * grad, rel=1e-12)


def test_nonfinite_raises_with_iteration():
    gs = _one([1.0, 2.0], [np.inf, 0.0])
    with pytest.raises(orc.OracleDivergence) as e:
        orc.apply_update(gs, hp(), lr=1.0, iteration=42)
    assert e.value.iteration == 42


# ---- test_cluster.py:93-105 aggregation ----
def test_all_reduce_kats():
    g = {"w": np.full((2, 2), 0.5)}
    assert np.array_equal(orc.all_reduce([dict(g) for _ in range(4)])["w"], np.full((2, 2), 2.0))
    x = np.random.default_rng(0).standard_normal((3, 3))
    assert np.all(orc.all_reduce([{"w": x}, {"w": -x}])["w"] == 0.0)
    with pytest.raises(ValueError, match="w"):
        orc.all_reduce([{"w": np.zeros(2)}, {"w": np.zeros(3)}])


# ---- golden vectors from the reference itself ----
MAN = manifest()


@pytest.mark.parametrize("case", MAN["cases"], ids=[c["name"] for c in MAN["cases"]])
def test_oracle_reproduces_reference_golden(case):
    arr = golden_arrays()
    w, m, lam, lr, it = run_oracle_case(case, MAN["hp"])
    assert np.array_equal(w, arr[case["name"] + "/w"])
    assert np.array_equal(m, arr[case["name"] + "/m"])
    assert np.array_equal(lam, arr[case["name"] + "/lambda"])
    assert lr == case["lr"]
    if "explicit_lr" not in case["extra"]:
        assert it == case["iteration_after"]


def test_oracle_schedule_golden():
    for hpn, mx, ipe, it, lr in MAN["schedule"]:
        assert orc.scheduled_lr(HP(**MAN["hp"][hpn]), it, mx, ipe) == lr


def test_oracle_divergence_golden():
    import gen
    from helpers import oracle_groups
    groups = oracle_groups(gen.RAGGED, 13)
    groups[2].grad[:] = np.inf  # b.weight
    with pytest.raises(orc.OracleDivergence) as e:
        orc.apply_update(groups, HP(**MAN["hp"]["plain"]), lr=1.0, iteration=42)
    assert e.value.iteration == MAN["divergence"]["iteration"]
    assert str(e.value) == MAN["divergence"]["message"]


def test_threaded_port_matches_oracle():
    from helpers import oracle_groups, LAYOUTS
    h = HP(**MAN["hp"]["lars_warm"])
    a = oracle_groups(LAYOUTS["mlp"], 5)
    b = [g.copy() for g in a]
    la = orc.apply_update(a, h, 0.3)
    port = orc.ThreadedPort(b, threads=4, block=1000)
    lb, ok = port.apply_update(h, 0.3)
    port.close()
    assert ok
    for ga, gb in zip(a, b):
        np.testing.assert_allclose(gb.param, ga.param, rtol=1e-13, atol=1e-16)
    for k in la:
        assert lb[k] == pytest.approx(la[k], rel=1e-12)
