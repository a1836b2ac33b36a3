"""Sharded RS -> LARS -> AG step on real GPUs (NCCL), world size 2 (and 4
when available): every rank ends with the same weights, equal to the
replicated oracle step within the one-step tolerance; 100 steps of the
sharded step match 100 single-GPU fused steps on the summed gradient (1e-4)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import gen
from helpers import HP, LAYOUTS, assert_params_close, oracle_groups
from oracle import lars_oracle as orc

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


HPKW = dict(base_lr=0.32, epochs=10, batch_size=512, warmup_epochs=2, lars_enabled=True)


def _worker(rank, world, port, layout_name, seed, steps, q, backend="nccl", max_iters=100):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_1709_05011_b200 import cluster, layouts, optim
    from paper_1709_05011_b200.flat import FlatParamSet
    layout = LAYOUTS.get(layout_name) or layouts.get(layout_name)
    hp = optim.HyperParams(**HPKW)
    st = optim.ScheduleState(max_iters, 10, 7)
    fps = FlatParamSet(layout, dev, world_size=world, rank=rank, symmetric=(backend == "p2p"))
    for grp, (w, _, m) in zip(fps, gen.group_inputs(layout, seed)):
        grp.param.copy_(torch.from_numpy(w))
        fps.set_momentum(grp.name, m)
    dp = cluster.DataParallelLars(fps, backend=backend)
    assert dp.backend == backend
    lams = None
    for t in range(steps):
        for grp, g in zip(fps, gen.step_grads(layout, seed * 31 + rank, t, g_scale=0.128)):
            grp.grad.copy_(torch.from_numpy(g))
        lams = dp.step(hp, st, grad_scale=1.0 / (256 * world), check=True)
    cluster.check_synchronized(fps)
    torch.cuda.synchronize()
    q.put((rank, fps.flat_param.cpu().numpy(), dict(lams), st.iteration))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, layout_name, seed, steps, backend="nccl", max_iters=100):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, layout_name, seed, steps, q, backend, max_iters))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _need(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")


@pytest.mark.parametrize("backend", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("layout_name", ["ragged", "mlp", "sweep:2e6:100"])
def test_sharded_step_matches_oracle(world, layout_name, backend, cuda):
    _need(world)
    from paper_1709_05011_b200 import layouts
    layout = LAYOUTS.get(layout_name) or layouts.get(layout_name)
    res = _run(world, layout_name, 5, 1, backend)
    for r in range(1, world):
        assert np.array_equal(res[r][1], res[0][1])
        assert res[r][2] == res[0][2]
    hp = HP(**HPKW)
    groups = oracle_groups(layout, 5)
    sets = [{grp.name: g.astype(np.float64) for grp, g in
             zip(groups, gen.step_grads(layout, 5 * 31 + r, 0, g_scale=0.128))} for r in range(world)]
    lam_ref, it = orc.dp_step([groups], sets, hp, 7, 100, 10, 256 * world)
    from paper_1709_05011_b200.flat import FlatParamSet
    ref_fps = FlatParamSet(layout, "cpu")
    w_got = np.concatenate([res[0][1][g.offset:g.offset + g.numel] for g in ref_fps])
    w_ref = np.concatenate([g.param.reshape(-1) for g in groups])
    assert_params_close(w_got, w_ref, layout, 1e-5, what="w")
    for k, v in lam_ref.items():
        assert res[0][2][k] == pytest.approx(v, rel=1e-6), k
    assert res[0][3] == it


@pytest.mark.parametrize("backend", ["nccl", "p2p"])
def test_sharded_trajectory_matches_single_gpu(backend, cuda):
    _need(2)
    world, steps, layout_name = 2, 100, "mlp"
    res = _run(world, layout_name, 9, steps, backend, max_iters=200)
    # single GPU: fused step on the summed gradient
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.flat import FlatParamSet
    layout = LAYOUTS[layout_name]
    fps = FlatParamSet(layout, cuda)
    for grp, (w, _, m) in zip(fps, gen.group_inputs(layout, 9)):
        grp.param.copy_(torch.from_numpy(w))
        grp.momentum_buf.copy_(torch.from_numpy(m))
    fps.invalidate_norm_cache()
    hp = optim.HyperParams(**HPKW)
    st = optim.ScheduleState(200, 10, 7)
    for t in range(steps):
        total = None
        for r in range(world):
            for grp, g in zip(fps, gen.step_grads(layout, 9 * 31 + r, t, g_scale=0.128)):
                grp.grad.copy_(torch.from_numpy(g))
            total = fps.flat_grad.clone() if total is None else total + fps.flat_grad
        fps.flat_grad.copy_(total)
        optim.sgd_step(fps, hp, st, grad_scale=1.0 / (256 * world))
    w1 = fps.flat_param.cpu().numpy()
    got = np.concatenate([res[0][1][g.offset:g.offset + g.numel] for g in fps])
    ref = np.concatenate([w1[g.offset:g.offset + g.numel] for g in fps])
    assert_params_close(got, ref, layout, 1e-4, what="w")


def _overlap_worker(rank, world, port, q):
    """Train a small conv net for 3 steps of 2 micro-batches twice: the plain
    p2p step and the backward-overlapped one (§8f1).  Same rank summation
    order -> bitwise identical weights."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    torch.backends.cudnn.deterministic = True  # bitwise-reproducible backward
    torch.backends.cudnn.benchmark = False
    from paper_1709_05011_b200 import optim
    from paper_1709_05011_b200.cluster import DataParallelLars
    from paper_1709_05011_b200.flat import FlatParamSet
    nn = torch.nn
    hp = optim.HyperParams(**HPKW)
    out = {}
    for mode in ("plain", "overlap"):
        torch.manual_seed(0)
        model = nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(),
                              nn.Conv2d(16, 32, 3, padding=1), nn.ReLU(), nn.Flatten(),
                              nn.Linear(32 * 8 * 8, 64), nn.ReLU(), nn.Linear(64, 10)).to(dev)
        fps = FlatParamSet.from_module(model, dev, world_size=world, rank=rank, symmetric=True)
        dp = DataParallelLars(fps, backend="p2p")
        ov = dp.overlap_backward(model, bucket_bytes=16 << 10) if mode == "overlap" else None
        if ov is not None:
            assert len(ov.buckets) > 2
        st = optim.ScheduleState(100, 10, 7)
        g = torch.Generator(device=dev)
        g.manual_seed(100 + rank)
        for _ in range(3):
            fps.zero_grads()
            for mb in range(2):
                x = torch.randn(8, 3, 8, 8, device=dev, generator=g)
                y = torch.randint(0, 10, (8,), device=dev, generator=g)
                loss = nn.functional.cross_entropy(model(x), y, reduction="sum")
                if ov is not None and mb == 1:
                    ov.arm()
                loss.backward()
            dp.step(hp, st, grad_scale=1.0 / (16 * world), check=True)
        torch.cuda.synchronize()
        out[mode] = fps.flat_param.cpu().numpy().copy()
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_backward_overlap_bitwise(world, cuda):
    _need(world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out = q.get(timeout=300)
        res[r] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        assert np.array_equal(res[r]["overlap"], res[r]["plain"]), r
        assert np.array_equal(res[r]["overlap"], res[0]["overlap"]), r
    assert np.isfinite(res[0]["plain"]).all()
