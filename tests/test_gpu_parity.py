"""GPU parity of the fused LARS step against the reference and the oracle.

Tolerances (BASELINE.json north star; form from SURVEY.md §8d):
  one step      |x_gpu - x_ref| <= 1e-5 |x_ref| + 1e-7 rms(layer)
  100 steps     same form at 1e-4
  lambda        |l_gpu - l_ref| <= 1e-6 |l_ref|
The GPU state is fp32, the reference fp64; inputs are fp32 values so both
start from identical numbers.
"""

import math

import numpy as np
import pytest
import torch

import gen
from helpers import (HP, LAYOUTS, assert_params_close, golden_arrays, manifest, oracle_groups,
                     run_oracle_case)
from oracle import lars_oracle as orc

pytestmark = pytest.mark.gpu

MAN = manifest()


def _optim():
    from paper_1709_05011_b200 import optim
    return optim


def load_fps(layout, seed, device, extra=None):
    from paper_1709_05011_b200.flat import FlatParamSet
    extra = extra or {}
    fps = FlatParamSet(layout, device)
    ins = gen.group_inputs(layout, seed, zero_w=tuple(extra.get("zero_w", ())),
                           zero_g=tuple(extra.get("zero_g", ())))
    for grp, (w, g, m) in zip(fps, ins):
        grp.param.copy_(torch.from_numpy(w))
        grp.grad.copy_(torch.from_numpy(g))
        grp.momentum_buf.copy_(torch.from_numpy(m))
    fps.invalidate_norm_cache()
    return fps


def flat_values(fps, which="param"):
    out = []
    for grp in fps:
        t = grp.param if which == "param" else grp.momentum_buf
        out.append(t.detach().double().cpu().numpy().reshape(-1))
    return np.concatenate(out)


def run_gpu_case(case, device):
    optim = _optim()
    layout = LAYOUTS[case["layout"]]
    hp = optim.HyperParams(**MAN["hp"][case["hp"]])
    extra = case["extra"]
    fps = load_fps(layout, case["seed"], device, extra)
    st = optim.ScheduleState(case["max_iters"], case["ipe"], case["iteration"])
    lams = None
    for t in range(case["steps"]):
        if t > 0:
            fps.set_grads({grp.name: g for grp, g in zip(fps, gen.step_grads(layout, case["seed"], t))})
        if "dp" in extra:
            from helpers import dp_grad_sets
            P, lb = extra["dp"], extra["local_batch"]
            total = None
            for gs in dp_grad_sets(layout, case["seed"], P, lb):
                fps.set_grads({grp.name: g for grp, g in zip(fps, gs)})
                total = fps.flat_grad.clone() if total is None else total + fps.flat_grad
            fps.flat_grad.copy_(total)
            lams = optim.sgd_step(fps, hp, st, grad_scale=1.0 / (P * lb))
        elif "explicit_lr" in extra:
            lams = optim.apply_update(fps, hp, extra["explicit_lr"], extra["iteration"])
        else:
            lams = optim.sgd_step(fps, hp, st)
    lam = np.array([lams[g.name] for g in fps])
    return fps, flat_values(fps), flat_values(fps, "m"), lam, st


@pytest.mark.parametrize("case", MAN["cases"], ids=[c["name"] for c in MAN["cases"]])
def test_step_matches_reference_golden(case, cuda):
    arr = golden_arrays()
    layout = LAYOUTS[case["layout"]]
    fps, w, m, lam, st = run_gpu_case(case, cuda)
    rtol = 1e-4 if case["steps"] > 1 else 1e-5
    assert_params_close(w, arr[case["name"] + "/w"], layout, rtol, what="w")
    assert_params_close(m, arr[case["name"] + "/m"], layout, rtol, what="m")
    ref_lam = arr[case["name"] + "/lambda"]
    np.testing.assert_allclose(lam, ref_lam, rtol=1e-6, atol=0)
    optim = _optim()
    lr, it, bad, status = optim.step_info(fps)
    assert bad == 2**31 - 1 and status == 0
    assert lr == pytest.approx(case["lr"], rel=1e-14, abs=0)
    if "explicit_lr" not in case["extra"]:
        assert st.iteration == case["iteration_after"]


@pytest.mark.parametrize("case", [c for c in MAN["cases"] if c["steps"] == 1],
                         ids=[c["name"] for c in MAN["cases"] if c["steps"] == 1])
def test_step_matches_oracle(case, cuda):
    layout = LAYOUTS[case["layout"]]
    w_ref, m_ref, lam_ref, _, _ = run_oracle_case(case, MAN["hp"])
    _, w, m, lam, _ = run_gpu_case(case, cuda)
    assert_params_close(w, w_ref, layout, 1e-5)
    assert_params_close(m, m_ref, layout, 1e-5)
    np.testing.assert_allclose(lam, lam_ref, rtol=1e-6, atol=0)


# ---- the reference KATs (pkg/tests/test_optim.py) through the GPU path ----

def _one_group(device, w, g, name="dense0.weight"):
    from paper_1709_05011_b200.flat import FlatParamSet
    w = np.asarray(w, np.float32)
    fps = FlatParamSet([(name, w.shape, "weight"), ("dense0.bias", (3,), "bias")], device)
    fps[name].param.copy_(torch.from_numpy(w))
    fps[name].grad.copy_(torch.from_numpy(np.asarray(g, np.float32)))
    fps.invalidate_norm_cache()
    return fps


def test_kat_lars_local_lr(cuda):
    optim = _optim()
    assert optim.lars_local_lr(np.array([1.0]), np.array([1.0]), 0.0, 0.001) == 0.001
    assert optim.lars_local_lr(np.zeros(4), np.ones(4), 0.0, 0.01) == 0.0
    assert optim.lars_local_lr(np.array([2.0]), np.array([1.0]), 0.5, 0.01) == pytest.approx(0.01, rel=1e-12)
    assert optim.lars_local_lr(np.array([3.0]), np.zeros(1), 0.0, 0.01) == 1.0
    w, g = np.array([3.0, 4.0]), np.array([1.0, 2.0])
    lam = optim.lars_local_lr(w, g, 0.0, 0.001)
    assert optim.lars_local_lr(4 * w, 4 * g, 0.0, 0.001) == pytest.approx(lam, rel=1e-12)


def test_kat_vanilla_step_exact(cuda):
    optim = _optim()
    rng = np.random.default_rng(5)
    w = rng.uniform(-1, 1, (2, 3)).astype(np.float32)
    fps = _one_group(cuda, w, np.full((2, 3), 0.25, np.float32))
    hp = optim.HyperParams(base_lr=1.0, epochs=10, batch_size=32, momentum=0.0, weight_decay=0.0)
    optim.apply_update(fps, hp, lr=1.0)
    got = fps["dense0.weight"].param.cpu().numpy()
    assert np.array_equal(got, (w.astype(np.float64) - 0.25).astype(np.float32))


def test_kat_momentum_two_steps(cuda):
    optim = _optim()
    w = np.array([[0.5, -1.0, 2.0], [0.25, 0.125, -0.75]], np.float32)
    fps = _one_group(cuda, w, np.full((2, 3), 0.5, np.float32))
    hp = optim.HyperParams(base_lr=0.1, epochs=10, batch_size=32, momentum=0.9, weight_decay=0.0)
    for _ in range(2):
        fps["dense0.weight"].grad.fill_(0.5)
        optim.apply_update(fps, hp, lr=0.1)
    got = fps["dense0.weight"].param.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(got, w - 0.1 * 0.5 * 2.9, rtol=1e-6)


def test_kat_lars_scales_update(cuda):
    optim = _optim()
    rng = np.random.default_rng(0)
    w = rng.uniform(-0.5, 0.5, (2, 3)).astype(np.float32)
    g = rng.standard_normal((2, 3)).astype(np.float32)
    fps = _one_group(cuda, w, g)
    hp = optim.HyperParams(base_lr=0.1, epochs=10, batch_size=32, momentum=0.0,
                           weight_decay=0.0, lars_enabled=True, lars_trust=0.02)
    lams = optim.apply_update(fps, hp, lr=0.1)
    w64, g64 = w.astype(np.float64), g.astype(np.float64)
    expect = 0.02 * np.linalg.norm(w64) / np.linalg.norm(g64) * 0.1 * g64
    got = fps["dense0.weight"].param.cpu().numpy().astype(np.float64)
    # the new weights to 1e-6; the step itself to fp32 resolution of w
    np.testing.assert_allclose(got, w64 - expect, rtol=1e-6)
    np.testing.assert_allclose(w64 - got, expect, rtol=0, atol=2 * np.spacing(np.float32(0.5)))
    assert lams["dense0.weight"] == pytest.approx(
        0.02 * np.linalg.norm(w64) / np.linalg.norm(g64), rel=1e-12)
    assert lams["dense0.bias"] == 1.0


def test_kat_lambda_one_reproduces_plain_step_bitwise(cuda):
    optim = _optim()
    outs = []
    for lars in (False, True):
        w = np.zeros((2, 3), np.float32)
        w[0, :2] = [3.0, 4.0]
        g = np.zeros((2, 3), np.float32)
        g[1, :2] = [4.0, 3.0]
        fps = _one_group(cuda, w, g)
        hp = optim.HyperParams(base_lr=0.1, epochs=10, batch_size=32, weight_decay=0.0,
                               lars_enabled=lars, lars_trust=1.0,
                               lars_skip_categories=frozenset({"bias"}))
        optim.apply_update(fps, hp, lr=0.1)
        outs.append(fps["dense0.weight"].param.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_kat_determinism_bitwise(cuda):
    optim = _optim()
    outs = []
    for _ in range(2):
        fps = load_fps(LAYOUTS["mlp"], 3, cuda)
        hp = optim.HyperParams(base_lr=0.3, epochs=10, batch_size=32, lars_enabled=True)
        st = optim.ScheduleState(10, 5)
        for _ in range(3):
            optim.sgd_step(fps, hp, st)
        outs.append(fps.flat_param.cpu().numpy().copy())
        assert st.iteration == 3
    assert np.array_equal(outs[0], outs[1])


def test_kat_divergence_raises_with_iteration(cuda):
    optim = _optim()
    from paper_1709_05011_b200.errors import DivergenceError
    fps = load_fps(gen.RAGGED, 13, cuda)
    fps["b.weight"].grad.fill_(float("inf"))
    hp = optim.HyperParams(**MAN["hp"]["plain"])
    with pytest.raises(DivergenceError) as e:
        optim.apply_update(fps, hp, lr=1.0, iteration=42)
    assert e.value.iteration == MAN["divergence"]["iteration"]
    assert str(e.value) == MAN["divergence"]["message"]


def test_kat_schedule_exhausted(cuda):
    optim = _optim()
    from paper_1709_05011_b200.errors import ScheduleExhaustedError
    fps = load_fps(gen.RAGGED, 1, cuda)
    before = fps.flat_param.clone()
    hp = optim.HyperParams(base_lr=0.1, epochs=10, batch_size=32)
    st = optim.ScheduleState(max_iterations=10, iterations_per_epoch=5, iteration=11)
    with pytest.raises(ScheduleExhaustedError):
        optim.sgd_step(fps, hp, st)
    assert torch.equal(before, fps.flat_param)
    assert st.iteration == 11


def test_device_schedule_matches_host(cuda):
    """The on-device lr (device_lr) equals scheduled_lr at every iteration."""
    optim = _optim()
    for hpn, mx, ipe, it, lr in MAN["schedule"]:
        fps = load_fps(gen.RAGGED, 1, cuda)
        hp = optim.HyperParams(**MAN["hp"][hpn])
        st = optim.ScheduleState(mx, ipe, it)
        optim.sgd_step(fps, hp, st, check=False)
        got = optim.step_info(fps)[0]
        assert got == pytest.approx(lr, rel=2e-16, abs=0), (hpn, it)


def test_device_exhaustion_flag(cuda):
    """In graph-style use the device refuses an exhausted step by itself."""
    optim = _optim()
    from paper_1709_05011_b200 import _native as nat
    fps = load_fps(gen.RAGGED, 1, cuda)
    before = fps.flat_param.clone()
    hp = optim.HyperParams(base_lr=0.1, epochs=10, batch_size=32)
    st = optim.ScheduleState(max_iterations=10, iterations_per_epoch=5, iteration=10)
    eng = fps.engine()
    eng.set_iteration(11)
    optim._launch_fused(fps, hp, st, lr=None, grad_scale=1.0, advance=True)
    lr, it, bad, status = eng.read_info()
    assert status == nat.LARS_STATUS_EXHAUSTED and it == 11
    assert torch.equal(before, fps.flat_param)
    assert int(eng.d_iter.item()) == 11


def test_reference_style_numpy_paramset(cuda):
    """apply_update on host numpy groups (the reference's own data type)."""
    optim = _optim()
    layout = gen.RAGGED
    hp_o = HP(**MAN["hp"]["lars_warm"])
    ref = oracle_groups(layout, 21)
    mine = [g.copy() for g in ref]
    lam_ref = orc.apply_update(ref, hp_o, 0.2, iteration=3)
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    lam = optim.apply_update(mine, hp, 0.2, iteration=3)
    assert set(lam) == set(lam_ref)
    for a, b in zip(mine, ref):
        # host arrays were updated in place (fp32 values)
        np.testing.assert_allclose(a.param, b.param, rtol=1e-5, atol=1e-7 * np.sqrt(np.mean(b.param ** 2)))
    for k in lam:
        assert lam[k] == pytest.approx(lam_ref[k], rel=1e-6)


# ---- full-size parameter sets (configs 2-5) ----

def _full_case(layout, device, seed, hp_kw, it=100, mx=3515, ipe=39, steps=1):
    optim = _optim()
    fps = load_fps(layout, seed, device)
    groups = oracle_groups(layout, seed)
    hp = optim.HyperParams(**hp_kw)
    hpo = HP(**hp_kw)
    st = optim.ScheduleState(mx, ipe, it)
    ito = it
    for t in range(steps):
        if t > 0:
            gs = gen.step_grads(layout, seed, t)
            fps.set_grads({grp.name: g for grp, g in zip(fps, gs)})
            for grp, g in zip(groups, gs):
                np.copyto(grp.grad, g.astype(np.float64))
        lams = optim.sgd_step(fps, hp, st)
        lam_ref, ito = orc.sgd_step(groups, hpo, ito, mx, ipe)
    w_ref = np.concatenate([g.param.reshape(-1) for g in groups])
    m_ref = np.concatenate([g.momentum_buf.reshape(-1) for g in groups])
    return fps, lams, w_ref, m_ref, lam_ref


BIG_HP = dict(base_lr=25.6, epochs=90, batch_size=32768, momentum=0.9, weight_decay=5e-4,
              poly_power=2.0, warmup_epochs=5, lars_enabled=True, lars_trust=1e-3)


@pytest.mark.parametrize("name", ["resnet50", "alexnet_bn"])
def test_full_size_one_step(name, cuda):
    from paper_1709_05011_b200 import layouts
    layout = layouts.get(name)
    fps, lams, w_ref, m_ref, lam_ref = _full_case(layout, cuda, 4, BIG_HP, it=300)
    assert_params_close(flat_values(fps), w_ref, layout, 1e-5, what="w")
    assert_params_close(flat_values(fps, "m"), m_ref, layout, 1e-5, what="m")
    for k, v in lam_ref.items():
        assert lams[k] == pytest.approx(v, rel=1e-6, abs=0), k


@pytest.mark.parametrize("spec", ["sweep:1e6:50", "sweep:4e6:300", "sweep:2e6:100",
                                  "sweep:2e6:1500"])  # (last: partials staged in the ring)
def test_sweep_layouts_three_steps(spec, cuda):
    from paper_1709_05011_b200 import layouts
    layout = layouts.get(spec)
    fps, lams, w_ref, m_ref, lam_ref = _full_case(layout, cuda, 9, BIG_HP, it=10, steps=3)
    # several steps of fp32 state: the multi-step tolerance
    assert_params_close(flat_values(fps), w_ref, layout, 1e-4, what="w")
    assert_params_close(flat_values(fps, "m"), m_ref, layout, 1e-4, what="m")
    for k, v in lam_ref.items():
        assert lams[k] == pytest.approx(v, rel=1e-6, abs=0), k


EMPTY_LAYOUT = [("head.weight", (0, 3), "weight"), ("a.weight", (3, 5), "weight"),
                ("mid.weight", (0,), "weight"), ("mid.bias", (0,), "bias"),
                ("one.bias", (1,), "bias"), ("b.weight", (129, 3), "weight"),
                ("tail.scale", (0,), "norm-scale")]


def test_zero_size_groups(cuda):
    """Groups with no elements at the start, middle and end (trusted and
    skipped): the oracle gives a trusted empty layer lambda 0 (its ||w|| is 0,
    optim.py:103-104) and leaves it alone; the neighbours update as usual."""
    fps, lams, w_ref, m_ref, lam_ref = _full_case(EMPTY_LAYOUT, cuda, 6, BIG_HP, it=10, steps=3)
    assert_params_close(flat_values(fps), w_ref, EMPTY_LAYOUT, 1e-4, what="w")
    assert_params_close(flat_values(fps, "m"), m_ref, EMPTY_LAYOUT, 1e-4, what="m")
    for k, v in lam_ref.items():
        assert lams[k] == pytest.approx(v, rel=1e-6, abs=0), k
    assert lams["head.weight"] == 0.0 and lams["mid.bias"] == 1.0
    optim = _optim()
    assert optim.step_info(fps)[2] == 2**31 - 1


def test_single_huge_layer(cuda):
    layout = [("fc6.weight", (4096, 9216), "weight"), ("fc6.bias", (4096,), "bias")]
    fps, lams, w_ref, m_ref, lam_ref = _full_case(layout, cuda, 2, BIG_HP)
    assert_params_close(flat_values(fps), w_ref, layout, 1e-5)
    assert lams["fc6.weight"] == pytest.approx(lam_ref["fc6.weight"], rel=1e-6, abs=0)


# ---- implementation properties ----

def _plan_step(fps, hp, st, grid, carry):
    """One fused launch through the C ABI with an explicit grid."""
    from paper_1709_05011_b200 import _native as nat
    from paper_1709_05011_b200.flat import _Plan, _ptr, _stream
    optim = _optim()
    eng = fps.engine()
    plan = _Plan(fps.segments(), len(fps), frozenset(hp.lars_skip_categories), grid=grid)
    ws = torch.empty(int(plan.info.workspace_bytes), dtype=torch.uint8, device=fps.device)
    nat.check(nat.load().lars_workspace_init(plan.handle, _ptr(ws), _stream()))
    flags = nat.LARS_STEP_ADVANCE_ITER
    h = optim.native_hparams(hp, st, flags=flags)
    nat.check(nat.load().lars_step(plan.handle, _ptr(fps.flat_param), _ptr(fps.flat_grad),
                                   _ptr(fps.momentum), nat.ctypes.byref(h), _ptr(eng.d_iter),
                                   _ptr(eng.d_sumsq), _ptr(eng.d_lambda), _ptr(eng.d_info),
                                   _ptr(ws), _stream()))
    return eng.d_lambda.clone()


@pytest.mark.parametrize("grid", [1, 7, 148, 296])
def test_grid_size_invariance(grid, cuda):
    from paper_1709_05011_b200 import layouts
    optim = _optim()
    layout = layouts.get("sweep:1e6:100")
    hp = optim.HyperParams(**BIG_HP)
    base = load_fps(layout, 3, cuda)
    st = optim.ScheduleState(3515, 39, 50)
    lam0 = None
    res = []
    for g in (0, grid):
        fps = load_fps(layout, 3, cuda)
        if g == 0:
            lam = optim.sgd_step(fps, hp, optim.ScheduleState(3515, 39, 50))
            lam = torch.tensor([lam[n] for n in fps.names()], dtype=torch.float64)
        else:
            fps.engine().set_iteration(50)
            lam = _plan_step(fps, hp, st, g, False).cpu()
        res.append((flat_values(fps), lam))
    assert_params_close(res[1][0], res[0][0], layout, 1e-6)
    torch.testing.assert_close(res[1][1], res[0][1], rtol=1e-13, atol=0)
    del base, lam0


def test_norm_carry_matches_fresh_norms(cuda):
    """Steps using the carried ||w||^2 agree with steps that re-read w."""
    optim = _optim()
    layout = LAYOUTS["mlp"]
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    a = load_fps(layout, 4, cuda)
    b = load_fps(layout, 4, cuda)
    sa, sb = optim.ScheduleState(200, 10), optim.ScheduleState(200, 10)
    for t in range(5):
        la = optim.sgd_step(a, hp, sa)              # carry used from step 2 on
        b.invalidate_norm_cache()
        lb = optim.sgd_step(b, hp, sb)              # always fresh
        for k in la:
            assert la[k] == pytest.approx(lb[k], rel=1e-13, abs=0)
    np.testing.assert_allclose(flat_values(a), flat_values(b), rtol=1e-6, atol=1e-9)


def test_external_write_invalidates_carry(cuda):
    optim = _optim()
    layout = LAYOUTS["mlp"]
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    key = frozenset(hp.lars_skip_categories)
    a = load_fps(layout, 4, cuda)
    st = optim.ScheduleState(200, 10)
    optim.sgd_step(a, hp, st)
    assert a.engine().carry_valid(key)
    a["dense0.weight"].param.mul_(3.0)               # bumps the shared version counter
    assert not a.engine().carry_valid(key)
    b = a.copy()                                     # fresh engine: norms re-read from w
    sb = optim.ScheduleState(200, 10, st.iteration)
    la = optim.sgd_step(a, hp, st)
    lb = optim.sgd_step(b, hp, sb)
    for k in la:
        assert la[k] == pytest.approx(lb[k], rel=1e-13, abs=0)


def test_split_form_equals_fused(cuda):
    """lars_partial_norms + lars_update == lars_step (P=1, nothing to reduce)."""
    optim = _optim()
    from paper_1709_05011_b200 import _native as nat
    from paper_1709_05011_b200.flat import _ptr, _stream
    layout = gen.RAGGED
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    a = load_fps(layout, 6, cuda)
    b = load_fps(layout, 6, cuda)
    optim.sgd_step(a, hp, optim.ScheduleState(100, 10, 7))
    eng = b.engine()
    eng.set_iteration(7)
    plan, ws = eng.plan(frozenset(hp.lars_skip_categories))
    h = optim.native_hparams(hp, optim.ScheduleState(100, 10, 7), flags=nat.LARS_STEP_ADVANCE_ITER)
    lib = nat.load()
    nat.check(lib.lars_partial_norms(plan.handle, _ptr(b.flat_param), _ptr(b.flat_grad),
                                     nat.ctypes.byref(h), _ptr(eng.d_iter), _ptr(eng.d_sumsq),
                                     _ptr(eng.d_info), _ptr(ws), _stream()))
    nat.check(lib.lars_update(plan.handle, _ptr(b.flat_param), _ptr(b.flat_grad),
                              _ptr(b.momentum), nat.ctypes.byref(h), _ptr(eng.d_sumsq),
                              _ptr(eng.d_lambda), _ptr(eng.d_info), _ptr(ws), _stream()))
    assert torch.equal(a.flat_param, b.flat_param)
    assert torch.equal(a.momentum, b.momentum)
    assert torch.equal(a.engine().d_lambda, eng.d_lambda)
    assert int(eng.d_iter.item()) == 8


def test_cuda_graph_replay(cuda):
    """The fused step (device lr + device iteration) replays from a CUDA graph."""
    optim = _optim()
    layout = LAYOUTS["mlp"]
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    a = load_fps(layout, 8, cuda)
    b = load_fps(layout, 8, cuda)
    sa = optim.ScheduleState(200, 10)
    for _ in range(4):
        optim.sgd_step(a, hp, sa)
    sb = optim.ScheduleState(200, 10)
    optim.sgd_step(b, hp, sb)                        # warm: plan, workspace, carry
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            optim._launch_fused(b, hp, sb, lr=None, grad_scale=1.0, advance=True)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(b.engine().d_iter.item()) == 4
    np.testing.assert_allclose(flat_values(b), flat_values(a), rtol=1e-6, atol=1e-9)


def test_padding_stays_zero(cuda):
    optim = _optim()
    fps = load_fps(gen.RAGGED, 2, cuda)
    hp = optim.HyperParams(**MAN["hp"]["lars_warm"])
    st = optim.ScheduleState(100, 10)
    for _ in range(3):
        optim.sgd_step(fps, hp, st)
    mask = torch.ones(fps.padded_numel, dtype=torch.bool, device=cuda)
    for g in fps:
        mask[g.offset:g.offset + g.numel] = False
    assert torch.count_nonzero(fps.flat_param[mask]) == 0
    assert torch.count_nonzero(fps.momentum[mask]) == 0
    assert math.isfinite(float(fps.flat_param.abs().max()))


def test_max_size_sweep_vs_torch_fp64(cuda):
    """Config 5 at its largest size: 1B parameters in 300 layers, one fused
    step against a plain PyTorch fp64 restatement of optim.py:98-108 (lambda)
    and :128-131 (update) on the GPU (the CPU oracle over all of it would
    need 24 GB), plus the oracle itself on nine sampled layers.

    Tolerance: the one-step form of the other tests for m (the kernel
    evaluates m = mu*m + (lam*lr)*s in fp64 and rounds it once), and for
    w = w - m the same plus 2^-23 |m|: w is updated in fp32 from the stored
    (rounded) m, so among 1e9 elements those where w and m cancel carry m's
    rounding, a representation error of the fp32 state."""
    from paper_1709_05011_b200 import layouts
    from paper_1709_05011_b200.flat import FlatParamSet
    optim = _optim()
    layout = layouts.get("sweep:1e9:300")
    fps = FlatParamSet(layout, cuda)
    gen_t = torch.Generator(device=cuda)
    gen_t.manual_seed(7)
    for grp in fps:
        grp.param.uniform_(-0.05, 0.05, generator=gen_t)
        grp.grad.normal_(0.0, 32.768, generator=gen_t)
        grp.momentum_buf.normal_(0.0, 1e-3, generator=gen_t)
    fps.invalidate_norm_cache()
    w0 = fps.flat_param.clone()
    m0 = fps.momentum.clone()
    hp = optim.HyperParams(**BIG_HP)
    st = optim.ScheduleState(3515, 39, 300)
    lr = optim.scheduled_lr(hp, st)
    scale = 1.0 / 32768
    lams = optim.sgd_step(fps, hp, st, grad_scale=scale)
    torch.cuda.synchronize()
    skip = set(hp.lars_skip_categories)
    for grp in fps:
        sl = slice(grp.offset, grp.offset + grp.numel)
        w = w0[sl].double()
        g = fps.flat_grad[sl].double() * scale
        m = m0[sl].double()
        if grp.category in skip:
            lam = 1.0
        else:
            wn = float(torch.linalg.vector_norm(w))
            gn = float(torch.linalg.vector_norm(g))
            denom = gn + hp.weight_decay * wn
            lam = 0.0 if wn == 0.0 else (1.0 if denom == 0.0 else hp.lars_trust * wn / denom)
        assert lams[grp.name] == pytest.approx(lam, rel=1e-6, abs=0), grp.name
        s = g + hp.weight_decay * w
        m_ref = hp.momentum * m + (lam * lr) * s
        w_ref = w - m_ref
        extra = {"m": torch.zeros_like(m_ref), "w": 2.0 ** -23 * m_ref.abs()}
        for got, ref, what in ((fps.flat_param[sl].double(), w_ref, "w"),
                               (fps.momentum[sl].double(), m_ref, "m")):
            rms = float(torch.sqrt(torch.mean(ref * ref)))
            tol = 1e-5 * ref.abs() + 1e-7 * rms + extra[what]
            bad = (got - ref).abs() > tol
            assert not bool(bad.any()), f"{what} {grp.name}: {int(bad.sum())} elements out of tolerance"
    # The oracle itself on a sample of the layers (a layer's update depends
    # only on its own w, g, m and the scalars, so sampled layers are checked
    # exactly as in the full set): first, last, largest and six spread ones.
    groups = list(fps)
    pick = {0, len(groups) - 1, max(range(len(groups)), key=lambda i: groups[i].numel)}
    pick |= {int(i) for i in np.linspace(1, len(groups) - 2, 6)}
    for i in sorted(pick):
        grp = groups[i]
        sl = slice(grp.offset, grp.offset + grp.numel)
        og = orc.Group(grp.name, w0[sl].double().cpu().numpy(),
                       fps.flat_grad[sl].double().cpu().numpy() * scale,
                       m0[sl].double().cpu().numpy(), grp.category)
        lam = orc.apply_update([og], hp, lr)[grp.name]
        assert lams[grp.name] == pytest.approx(lam, rel=1e-6, abs=0), grp.name
        w_ref, m_ref = og.param, og.momentum_buf
        for got, ref, extra, what in (
                (fps.flat_param[sl].double().cpu().numpy(), w_ref, 2.0 ** -23 * np.abs(m_ref), "w"),
                (fps.momentum[sl].double().cpu().numpy(), m_ref, 0.0, "m")):
            rms = float(np.sqrt(np.mean(ref * ref)))
            bad = np.abs(got - ref) > 1e-5 * np.abs(ref) + 1e-7 * rms + extra
            assert not bad.any(), f"oracle {what} {grp.name}: {int(bad.sum())} elements out of tolerance"


def test_norm_carry_many_chunks_per_warp(cuda):
    """A set large enough that the CTAs owning the tapered 1-batch chunks have
    several rounds (> 256 chunks per warp) of carried sums to fold: carried
    ||w||^2 must match a fresh re-read of w."""
    from paper_1709_05011_b200 import layouts
    from paper_1709_05011_b200.flat import FlatParamSet
    optim = _optim()
    layout = layouts.get("sweep:128e6:50")
    sets = []
    for _ in range(2):
        fps = FlatParamSet(layout, cuda)
        g = torch.Generator(device=cuda)
        g.manual_seed(3)
        for grp in fps:
            grp.param.uniform_(-0.05, 0.05, generator=g)
        fps.invalidate_norm_cache()
        sets.append(fps)
    a, b = sets
    info = a.engine().plan(frozenset(optim.HyperParams(**BIG_HP).lars_skip_categories))[0].info
    # the last CTAs' ranges are all 1-batch chunks: > 256 per warp
    assert info.nbatches / info.grid / 8 > 256
    hp = optim.HyperParams(**BIG_HP)
    sa, sb = optim.ScheduleState(3515, 39, 300), optim.ScheduleState(3515, 39, 300)
    for t in range(3):
        for fps in (a, b):
            g = torch.Generator(device=cuda)
            g.manual_seed(100 + t)
            fps.flat_grad.normal_(0.0, 32.0, generator=g)
        la = optim.sgd_step(a, hp, sa, grad_scale=1.0 / 32768)    # carry from step 2 on
        b.invalidate_norm_cache()
        lb = optim.sgd_step(b, hp, sb, grad_scale=1.0 / 32768)    # always fresh
        for k in la:
            assert la[k] == pytest.approx(lb[k], rel=1e-12, abs=0), (t, k)
    assert torch.allclose(a.flat_param, b.flat_param, rtol=1e-6, atol=1e-9)


def test_plans_of_different_sizes_interleaved(cuda):
    """A plan created after a larger one (smaller shared-memory footprint)
    must not break the larger plan's next launch: the kernels' dynamic
    shared-memory limit is only ever raised (regression: the host ParamSet
    pipeline runs several plans in turn)."""
    from paper_1709_05011_b200 import layouts
    optim = _optim()
    big = load_fps(layouts.get("resnet50"), 3, cuda)
    small = load_fps(LAYOUTS["ragged"], 3, cuda)
    hp = optim.HyperParams(**BIG_HP)
    for fps in (big, small, big, small, big):
        optim.apply_update(fps, hp, 0.01, iteration=1)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(big.flat_param).all()) and bool(torch.isfinite(small.flat_param).all())
