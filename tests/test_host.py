"""CPU tests of the host side: optimizer API surface, layouts, flat storage,
the C ABI library (load, exports, host-only planning, error codes) and the
benchmark's reference arm.  No CUDA calls are made."""

import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_1709_05011_b200 import _native as nat, layouts, optim
from paper_1709_05011_b200.errors import ConfigError, ScheduleExhaustedError
from paper_1709_05011_b200.flat import ALIGN, FlatParamSet, _Plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- optimizer API (pkg/tests/test_optim.py KATs on the host functions) ----

def make_hp(**kw):
    base = dict(base_lr=0.1, epochs=10, batch_size=32)
    base.update(kw)
    return optim.HyperParams(**base)


def test_linear_scaling_and_budget():
    assert optim.linear_scaled_lr(0.02, 512, 4096) == 0.16
    assert optim.linear_scaled_lr(0.2, 256, 32768) == 25.6
    with pytest.raises(ConfigError):
        optim.linear_scaled_lr(0.1, 0, 64)
    assert optim.max_iterations(50, 9000, 32) == 14062
    assert optim.max_iterations(1, 64, 64) == 1


def test_schedule_contract():
    hp = make_hp(base_lr=0.4, poly_power=2.0, warmup_epochs=2)
    st = optim.ScheduleState(max_iterations=100, iterations_per_epoch=10)
    st.iteration = 0
    assert optim.scheduled_lr(hp, st) == pytest.approx(0.4 / 20)
    st.iteration = 19
    assert optim.scheduled_lr(hp, st) == 0.4
    st.iteration = 20
    assert optim.scheduled_lr(hp, st) == 0.4
    st.iteration = 100
    assert optim.scheduled_lr(hp, st) == 0.0
    st.iteration = 101
    with pytest.raises(ScheduleExhaustedError):
        optim.scheduled_lr(hp, st)
    rows = optim.schedule_table(make_hp(base_lr=0.4), optim.ScheduleState(10, 5))
    assert len(rows) == 10 and rows[0] == (0, 0.4)


@pytest.mark.parametrize("kw", [dict(base_lr=-1.0), dict(momentum=1.0), dict(warmup_epochs=10),
                                dict(weight_decay=-1e-4), dict(poly_power=0.0),
                                dict(lars_trust=0.0), dict(base_lr=float("inf"))])
def test_hyperparam_validation(kw):
    with pytest.raises(ConfigError):
        make_hp(**kw)


def test_schedule_state_validation():
    with pytest.raises(ConfigError):
        optim.ScheduleState(0, 10)


def test_native_hparams_packing():
    hp = make_hp(base_lr=25.6, warmup_epochs=5, lars_enabled=True, lars_trust=2e-3)
    st = optim.ScheduleState(3515, 39)
    h = optim.native_hparams(hp, st, grad_scale=1 / 32768, flags=nat.LARS_STEP_ADVANCE_ITER)
    assert h.warmup_iters == 195 and h.max_iters == 3515 and h.lars_enabled == 1
    assert h.trust == 2e-3 and h.grad_scale == 1 / 32768
    assert h.flags == nat.LARS_STEP_ADVANCE_ITER
    h = optim.native_hparams(hp, None, lr=0.5)
    assert h.flags & nat.LARS_STEP_EXPLICIT_LR and h.lr == 0.5


def test_lambda_from_sums_matches_reference_formula():
    assert optim.lambda_from_sums(1.0, 1.0, 0.0, 0.001) == 0.001
    assert optim.lambda_from_sums(0.0, 4.0, 0.0, 0.01) == 0.0
    assert optim.lambda_from_sums(4.0, 1.0, 0.5, 0.01) == pytest.approx(0.01, rel=1e-12)
    assert optim.lambda_from_sums(9.0, 0.0, 0.0, 0.01) == 1.0


# ---- layouts ----

def test_layout_sizes():
    assert layouts.total_params(layouts.resnet50()) == 25_557_032
    assert len(layouts.resnet50()) == 161
    assert layouts.total_params(layouts.alexnet_bn()) == 61_103_144
    assert len(layouts.alexnet_bn()) == 26
    assert layouts.total_params(layouts.mlp()) == 26_634
    assert layouts.total_params(layouts.lenet5()) == 61_706
    cats = [c for _, _, c in layouts.resnet50()]
    assert cats.count("weight") == 54 and cats.count("norm-scale") == 53
    sw = layouts.sweep(1_000_000, 50)
    assert len(sw) == 50 and all(n[1][0] % 32 == 0 and n[1][0] >= 64 for n in sw)


def test_resnet50_layout_matches_torchvision():
    tv = pytest.importorskip("torchvision")
    model = tv.models.resnet50(weights=None)
    fps = FlatParamSet.from_module(model, "cpu")
    assert [(n, s, c) for n, s, c in fps.layout] == [(n, tuple(s), c) for n, s, c in layouts.resnet50()]


# ---- flat storage (nn.ParamSet surface) ----

def test_flat_layout_and_views():
    fps = FlatParamSet(layouts.mlp(), "cpu")
    assert fps.numel == 26_634
    for g in fps:
        assert g.offset % ALIGN == 0
        assert g.param.data_ptr() == fps.flat_param.data_ptr() + 4 * g.offset
        assert g.param.shape == g.shape and g.momentum_buf is not None
    assert fps.padded_numel % ALIGN == 0
    fps["dense0.weight"].param.fill_(2.0)
    assert float(fps.flat_param[fps["dense0.weight"].offset]) == 2.0
    with pytest.raises(ConfigError):
        FlatParamSet([("a", (2,), "weight"), ("a", (3,), "bias")], "cpu")


def test_set_grads_copy_checksum():
    layout = layouts.lenet5()
    fps = FlatParamSet(layout, "cpu")
    grads = {n: np.full(s, 0.5, np.float32) for n, s, _ in layout}
    fps.set_grads(grads)
    assert float(fps["fc1.weight"].grad.mean()) == 0.5
    flat = torch.arange(fps.padded_numel, dtype=torch.float32)
    fps.set_grads(flat)
    assert torch.equal(fps.flat_grad, flat)
    c1 = fps.checksum()
    twin = fps.copy()
    assert twin.checksum() == c1 and twin.flat_param.data_ptr() != fps.flat_param.data_ptr()
    twin["conv1.weight"].param[0, 0, 0, 0] += 1.0
    assert twin.checksum() != c1
    fps.zero_grads()
    assert float(fps.flat_grad.abs().sum()) == 0.0


def test_from_module_binds_parameters_and_categories():
    m = torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3), torch.nn.BatchNorm2d(4), torch.nn.ReLU(),
                            torch.nn.Flatten(), torch.nn.Linear(4 * 6 * 6, 5))
    before = [p.detach().clone() for p in m.parameters()]
    fps = FlatParamSet.from_module(m, "cpu")
    cats = dict((n, c) for n, _, c in fps.layout)
    assert cats == {"0.weight": "weight", "0.bias": "bias", "1.weight": "norm-scale",
                    "1.bias": "norm-shift", "4.weight": "weight", "4.bias": "bias"}
    for p, b in zip(m.parameters(), before):
        assert torch.equal(p.detach(), b)
    # backward accumulates straight into the flat gradient
    x = torch.randn(2, 3, 8, 8)
    m(x).sum().backward()
    assert float(fps.flat_grad.abs().sum()) > 0
    assert fps["4.bias"].grad.data_ptr() == m[4].bias.grad.data_ptr()


def test_sharded_momentum_helpers():
    layout = layouts.mlp()
    full = FlatParamSet(layout, "cpu")
    seen = {}
    for r in range(4):
        fps = FlatParamSet(layout, "cpu", world_size=4, rank=r)
        for g in fps:
            vals = np.arange(g.numel, dtype=np.float32) + 1000 * g.index
            fps.set_momentum(g.name, vals)
            part = fps.get_momentum(g.name)
            if part is not None:
                sl = fps.shard_slices(g.name)[1]
                seen.setdefault(g.name, []).append((sl.start, part.numpy().copy()))
    for g in full:
        got = np.concatenate([p for _, p in sorted(seen[g.name], key=lambda t: t[0])])
        assert np.array_equal(got, np.arange(g.numel, dtype=np.float32) + 1000 * g.index)


# ---- the C ABI library ----

def test_library_exports_every_header_symbol():
    lib = nat.load()
    with open(os.path.join(ROOT, "include", "lars_b200.h")) as f:
        declared = re.findall(r"LARS_API\s+[\w\s\*]+?\b(lars_\w+)\s*\(", f.read())
    assert set(declared) == set(nat.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.lars_abi_version() == 1
    assert lib.lars_strerror(0) == b"ok"
    assert b"misaligned" in lib.lars_strerror(nat.ctypes.c_int(2))
    # no symbol beyond the ABI leaks out (visibility=hidden)
    out = subprocess.run(["nm", "-D", "--defined-only", nat.lib_path()], capture_output=True, text=True)
    if out.returncode == 0:
        exported = {l.split()[-1] for l in out.stdout.splitlines() if " T " in l}
        assert exported == set(declared)


def _host_plan(segs, nlayers, grid=296):
    return _Plan(segs, nlayers, frozenset(), grid=grid, host_only=True)


@pytest.mark.parametrize("name,grid", [("resnet50", 296), ("alexnet_bn", 296), ("mlp", 7),
                                       ("sweep:4e6:300", 296), ("mlp", 1)])
def test_host_plan_partition_invariants(name, grid):
    fps = FlatParamSet(layouts.get(name), "cpu")
    plan = _host_plan(fps.segments(), len(fps), grid)
    info = plan.info
    assert info.grid == grid and info.threads == 256
    assert info.elements == sum(ln for _, ln, _, _ in fps.segments())
    assert info.nbatches == sum((ln // 4 + 31) // 32 for _, ln, _, _ in fps.segments())
    wb0 = np.zeros(grid * 8 + 1, np.int64)
    ps = np.zeros(info.npieces, np.int32)
    pc = np.zeros(info.npieces, np.int32)
    nat.check(nat.load().lars_plan_partition(plan.handle, wb0.ctypes.data, ps.ctypes.data,
                                             pc.ctypes.data))
    assert wb0[0] == 0 and wb0[-1] == info.nbatches and np.all(np.diff(wb0) >= 0)
    # pieces are (CTA, segment) pairs in buffer order; every segment is covered
    assert np.all(np.diff(pc) >= 0)
    assert set(ps.tolist()) == set(range(info.nseg))
    assert info.workspace_bytes > 0 and info.smem_bytes < 227 * 1024


@pytest.mark.parametrize("name", ["resnet50", "alexnet_bn", "mlp", "sweep:1e6:300"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_tile_the_buffer_and_plan(name, world):
    """Host side of the P-rank step (up to LARS_MAX_RANKS = 8): equal aligned
    shards, every element of every group in exactly one shard's segment
    table, and a launch plan for every rank's shard."""
    layout = layouts.get(name)
    full = FlatParamSet(layout, "cpu")
    covered = {g.name: np.zeros(g.numel, np.int32) for g in full}
    for r in range(world):
        fps = FlatParamSet(layout, "cpu", world_size=world, rank=r)
        assert fps.padded_numel % (32 * world) == 0
        assert fps.shard_numel * world == fps.padded_numel
        assert fps.shard_lo == r * fps.shard_numel
        segs = fps.segments()
        assert len(segs) == len(fps)
        for g, (off, ln, layer, _) in zip(fps, segs):
            assert layer == g.index
            assert off % 4 == 0 and ln % 4 == 0
            if ln:
                lo = fps.shard_lo + off - g.offset
                covered[g.name][lo:min(lo + ln, g.numel)] += 1
        plan = _host_plan(segs, len(fps), 296)
        assert plan.info.elements == sum(ln for _, ln, _, _ in segs) <= fps.shard_numel
    for name_, c in covered.items():
        assert np.all(c == 1), name_


def test_plan_error_codes():
    lib = nat.load()

    def create(segs, nlayers=2, grid=4, flags=nat.LARS_PLAN_HOST_ONLY):
        arr = (nat.Segment * max(1, len(segs)))()
        for i, (o, n, l) in enumerate(segs):
            arr[i].offset, arr[i].length, arr[i].layer, arr[i].flags = o, n, l, 1
        h = ctypes.c_void_p()
        rc = lib.lars_plan_create(arr, len(segs), nlayers, grid, flags, ctypes.byref(h))
        if rc == 0:
            lib.lars_plan_destroy(h)
        return rc

    assert create([(0, 64, 0), (64, 32, 1)]) == nat.LARS_OK
    assert create([(0, 62, 0)]) == nat.LARS_ERR_ALIGNMENT
    assert create([(0, 64, 0), (32, 32, 1)]) == nat.LARS_ERR_LAYOUT  # overlap
    assert create([(0, 64, 5)]) == nat.LARS_ERR_INVALID              # layer id
    assert create([(0, 64, 0)], grid=0) == nat.LARS_ERR_INVALID      # host-only needs a grid
    assert create([]) == nat.LARS_OK             # empty set is valid


def test_host_only_plan_refuses_launch():
    lib = nat.load()
    fps = FlatParamSet(layouts.mlp(), "cpu")
    plan = _host_plan(fps.segments(), len(fps), 4)
    h = optim.native_hparams(make_hp(), optim.ScheduleState(10, 5))
    z = ctypes.c_void_p(16)
    rc = lib.lars_step(plan.handle, z, z, z, ctypes.byref(h), z, None, None, z, z, None)
    assert rc == nat.LARS_ERR_HOST_ONLY_PLAN
    assert lib.lars_workspace_init(plan.handle, z, None) == nat.LARS_ERR_HOST_ONLY_PLAN


# ---- benchmark reference arm (CPU only) ----

def test_bench_reference_arm_prints_contract_line():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--workload", "mlp"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    stock = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "batchlab"))
    assert line["cpu_baseline"]["kind"] == ("reference" if stock else "port")
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["steps"] == 2


def test_bench_reference_arm_dp_sample_rank0_only():
    """N>1: rank 0 times the reference DP step (all_reduce + /B + P x update)
    on a 1/P sample; other ranks print nothing and exit 0."""
    for rank, expect_line in ((0, True), (1, False)):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2")
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                              "--gpus", "2", "--steps", "2", "--warmup", "1", "--workload", "mlp"],
                             capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-2000:]
        if expect_line:
            line = json.loads(out.stdout.strip().splitlines()[-1])
            assert line["n_gpus"] == 2 and "all_reduce" in line["cpu_baseline"]["sample"]
        else:
            assert out.stdout.strip() == ""


def test_alexnet_bn_module_matches_layout():
    from paper_1709_05011_b200.train import alexnet_bn
    fps = FlatParamSet.from_module(alexnet_bn(), "cpu")
    assert [(n, s, c) for n, s, c in fps.layout] == [(n, tuple(s), c) for n, s, c in layouts.alexnet_bn()]


# ---- cluster.all_reduce (pkg/tests/test_cluster.py:92-105 restated) ----

def test_all_reduce_identical_summands():
    from paper_1709_05011_b200 import cluster
    g = {"w": np.full((2, 2), 0.5)}
    out = cluster.all_reduce([dict(g) for _ in range(4)])
    assert np.array_equal(out["w"], np.full((2, 2), 2.0))


def test_all_reduce_cancellation_is_exact():
    from paper_1709_05011_b200 import cluster
    g = np.random.default_rng(0).standard_normal((3, 3))
    out = cluster.all_reduce([{"w": g}, {"w": -g}])
    assert np.all(out["w"] == 0.0)


def test_all_reduce_shape_mismatch_names_group():
    from paper_1709_05011_b200 import cluster
    from paper_1709_05011_b200.errors import ProtocolError
    with pytest.raises(ProtocolError, match="'w'"):
        cluster.all_reduce([{"w": np.zeros(2)}, {"w": np.zeros(3)}])
    with pytest.raises(ProtocolError, match="worker 2"):
        cluster.all_reduce([{"w": np.zeros(2)}, {"w": np.zeros(2)}, {"v": np.zeros(2)}])


def test_all_reduce_pairwise_left_tree_order():
    """reduction.py:30-47: ((a+b)+(c+d))+e -- visible in fp64 rounding."""
    from paper_1709_05011_b200 import cluster
    vals = [1e16, 1.0, -1e16, 1.0, 3.0]
    out = cluster.all_reduce([{"x": np.array([v])} for v in vals])
    expect = ((vals[0] + vals[1]) + (vals[2] + vals[3])) + vals[4]
    assert out["x"][0] == expect
    assert out["x"][0] == orc_all_reduce([{"x": np.array([v])} for v in vals])["x"][0]


def orc_all_reduce(sets):
    from oracle import lars_oracle as orc
    return orc.all_reduce(sets)


@pytest.mark.parametrize("name", ["resnet50", "alexnet_bn", "mlp"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shared_flags_mark_layers_cut_by_shard_edges(name, world):
    """FlatParamSet.shared_flags (LARS_SEG_SHARED for the streamed sharded
    step): a group is shared iff it has elements in this shard AND in
    another one; every cut group is shared on every rank that holds part
    of it, and at most two groups per shard are shared (its first / last)."""
    layout = layouts.get(name)
    holders = {}
    for r in range(world):
        fps = FlatParamSet(layout, "cpu", world_size=world, rank=r)
        flags = fps.shared_flags()
        assert len(flags) == len(fps.groups)
        assert sum(flags) <= 2
        for g, f, (off, ln, _, _) in zip(fps.groups, flags, fps.segments()):
            if ln > 0:
                holders.setdefault(g.name, []).append((r, f))
            else:
                assert not f
    for gname, hs in holders.items():
        shared = len(hs) > 1
        assert all(f == shared for _, f in hs), gname


@pytest.mark.parametrize("name", ["resnet50", "alexnet_bn", "sweep:1e6:50", "sweep:16e6:100"])
def test_plan_keeps_two_ctas_per_sm(name):
    """Shared-memory budget: the config plans must fit two CTAs per SM
    (228 KiB per SM, 1 KiB reserved per CTA).  A few hundred bytes more per
    CTA halve the resident grid and cost ~40 % of the step (measured)."""
    layout = layouts.get(name)
    fps = FlatParamSet(layout, "cpu")
    plan = _Plan(fps.segments(), len(fps), frozenset(optim.DEFAULT_LARS_SKIP), grid=296,
                 host_only=True)
    assert plan.info.smem_bytes <= (228 * 1024) // 2 - 1024, plan.info.smem_bytes


def test_host_mirror_parts_split():
    """The host ParamSet pipeline's parts: contiguous runs of whole groups,
    roughly equal element counts, at most MAX_PARTS, none empty."""
    from paper_1709_05011_b200 import hostset, layouts
    for lay in (layouts.get("resnet50"), layouts.get("alexnet_bn"), layouts.mlp()):
        numels = [int(np.prod(s)) for _, s, _ in lay]
        parts = hostset._split(numels, hostset.PART_MIN_ELEMS, hostset.MAX_PARTS)
        assert parts[0][0] == 0 and parts[-1][1] == len(numels)
        assert all(a < b for a, b in parts)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(len(parts) - 1))
        assert len(parts) <= hostset.MAX_PARTS
    assert len(hostset._split([10] * 5, 1, 8)) == 5
    assert hostset._split([100], 1, 8) == [(0, 1)]
    r50 = [int(np.prod(s)) for _, s, _ in layouts.get("resnet50")]
    assert len(hostset._split(r50, hostset.PART_MIN_ELEMS, hostset.MAX_PARTS)) == 6
