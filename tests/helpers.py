"""Shared test helpers: golden fixtures, oracle runs, tolerance checks."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(HERE, "golden"))

import gen  # noqa: E402
from oracle import lars_oracle as orc  # noqa: E402
from paper_1709_05011_b200 import layouts  # noqa: E402

GOLDEN_DIR = os.path.join(HERE, "golden")
LAYOUTS = {"ragged": gen.RAGGED, "mlp": layouts.mlp(), "lenet5": layouts.lenet5()}


def manifest():
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
        return json.load(f)


def golden_arrays():
    return np.load(os.path.join(GOLDEN_DIR, "lars_golden.npz"))


class HP:
    """Duck-typed HyperParams for the oracle."""

    def __init__(self, **kw):
        self.base_lr = kw["base_lr"]
        self.epochs = kw.get("epochs", 10)
        self.batch_size = kw.get("batch_size", 32)
        self.momentum = kw.get("momentum", 0.9)
        self.weight_decay = kw.get("weight_decay", 5e-4)
        self.poly_power = kw.get("poly_power", 2.0)
        self.warmup_epochs = kw.get("warmup_epochs", 0)
        self.lars_enabled = kw.get("lars_enabled", False)
        self.lars_trust = kw.get("lars_trust", 1e-3)
        self.lars_skip_categories = kw.get("lars_skip_categories", orc.DEFAULT_LARS_SKIP)


def oracle_groups(layout, seed, extra=None):
    extra = extra or {}
    ins = gen.group_inputs(layout, seed, zero_w=tuple(extra.get("zero_w", ())),
                           zero_g=tuple(extra.get("zero_g", ())))
    return [orc.Group(n, w.astype(np.float64), g.astype(np.float64), m.astype(np.float64), c)
            for (n, _, c), (w, g, m) in zip(layout, ins)]


def dp_grad_sets(layout, seed, P, local_batch):
    return [[g for g in gen.step_grads(layout, seed * 31 + r, 0, g_scale=1e-3 * local_batch)]
            for r in range(P)]


def run_oracle_case(case, hp_table):
    """Replay one golden case on the oracle; returns (w, m, lambdas, lr, it)."""
    layout = LAYOUTS[case["layout"]]
    hp = HP(**hp_table[case["hp"]])
    extra = case["extra"]
    groups = oracle_groups(layout, case["seed"], extra)
    it = case["iteration"]
    lams, lr = None, None
    for t in range(case["steps"]):
        if t > 0:
            for grp, g in zip(groups, gen.step_grads(layout, case["seed"], t)):
                np.copyto(grp.grad, g.astype(np.float64))
        if "dp" in extra:
            P, lb = extra["dp"], extra["local_batch"]
            sets = [{grp.name: g.astype(np.float64) for grp, g in zip(groups, gs)}
                    for gs in dp_grad_sets(layout, case["seed"], P, lb)]
            lr = orc.scheduled_lr(hp, it, case["max_iters"], case["ipe"])
            lams, it = orc.dp_step([groups], sets, hp, it, case["max_iters"], case["ipe"], P * lb)
        elif "explicit_lr" in extra:
            lr = extra["explicit_lr"]
            lams = orc.apply_update(groups, hp, lr, iteration=extra["iteration"])
        else:
            lr = orc.scheduled_lr(hp, it, case["max_iters"], case["ipe"])
            lams, it = orc.sgd_step(groups, hp, it, case["max_iters"], case["ipe"])
    w = np.concatenate([g.param.reshape(-1) for g in groups])
    m = np.concatenate([g.momentum_buf.reshape(-1) for g in groups])
    lam = np.array([lams[g.name] for g in groups])
    return w, m, lam, lr, it


def group_slices(layout):
    out, o = [], 0
    for n in gen.layout_numel(layout):
        out.append(slice(o, o + n))
        o += n
    return out


def assert_params_close(got, ref, layout, rtol, floor=None, what="param"):
    """Per-element |got-ref| <= rtol*|ref| + floor*rms(layer);
    the absolute floor covers elements that cancel to ~0.  The floor scales
    with the tolerance: 1e-7 at rtol 1e-5 (one step), 1e-6 at rtol 1e-4
    (100 steps of fp32 state against the fp64 reference)."""
    if floor is None:
        floor = 1e-2 * rtol
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape
    worst = 0.0
    for (name, _, _), sl in zip(layout, group_slices(layout)):
        r = ref[sl]
        g = got[sl]
        rms = float(np.sqrt(np.mean(r * r))) if r.size else 0.0
        tol = rtol * np.abs(r) + floor * rms
        err = np.abs(g - r)
        bad = err > tol
        if np.any(bad):
            i = int(np.argmax(err - tol))
            raise AssertionError(
                f"{what} {name}[{i}]: got {g[i]!r} ref {r[i]!r} err {err[i]:.3e} tol {tol[i]:.3e}")
        if r.size:
            worst = max(worst, float(np.max(err / np.maximum(tol, 1e-300))))
    return worst


def rolled_grads(base, t):
    """Fresh gradients for step t of a long trajectory, cheap at 61M params:
    every group of the base set rolled by a step-dependent offset and scaled
    by a signed power of two (exact in fp32, so device and oracle see the same
    numbers)."""
    s = np.float32((-1.0) ** t * 2.0 ** ((t % 3) - 1))
    return [(np.roll(b.reshape(-1), 7919 * t + 13 * i) * s).reshape(b.shape)
            for i, b in enumerate(base)]


def free_port():
    """A rendezvous port below the kernel's ephemeral range (32768-60999 on
    Linux), so that no outgoing connection of another process can take it
    between this check and the TCPStore's bind."""
    import random
    import socket
    for _ in range(200):
        port = random.randrange(20000, 32000)
        with socket.socket() as s:
            try:
                s.bind(("127.0.0.1", port))
            except OSError:
                continue
            return port
    raise RuntimeError("no free rendezvous port")


def spawn_ranks(target, world, args_of_port, timeout=600, attempts=3):
    """Start `world` spawned processes target(rank, world, port, *args) and
    collect one queue message per rank; a rendezvous that fails to bind its
    port (EADDRINUSE) is retried on another port.  Fails fast when a rank
    dies without reporting.  Returns the messages by rank."""
    import queue as _queue
    import time
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    for attempt in range(attempts):
        q = ctx.Queue()
        port = free_port()
        procs = [ctx.Process(target=target, args=(r, world, port, q, *args_of_port))
                 for r in range(world)]
        for p in procs:
            p.start()
        res, deadline, retry = {}, time.monotonic() + timeout, False
        try:
            while len(res) < world:
                try:
                    r = q.get(timeout=2)
                except _queue.Empty:
                    dead = [p for p in procs if p.exitcode not in (None, 0)]
                    if dead:
                        raise AssertionError(f"rank process exited with {dead[0].exitcode}")
                    if time.monotonic() > deadline:
                        raise AssertionError("ranks did not report in time")
                    continue
                if r[0] == "init-failed":
                    if "EADDRINUSE" in r[2] or "address already in use" in r[2]:
                        retry = True
                        break
                    raise AssertionError(f"rank {r[1]} failed to initialise: {r[2]}")
                res[r[0]] = r
        finally:
            if retry or len(res) < world:
                for p in procs:
                    if p.is_alive():
                        p.kill()
            for p in procs:
                p.join(timeout=120)
        if retry and attempt + 1 < attempts:
            continue
        assert not retry, "rendezvous port kept colliding"
        for p in procs:
            assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
        return res
    raise AssertionError("unreachable")


def init_group(backend, rank, world, port, q, device_id=None):
    """init_process_group for a spawned rank; a failure is reported on `q`
    (so spawn_ranks can retry a port collision) and re-raised."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        if device_id is None:
            dist.init_process_group(backend, rank=rank, world_size=world)
        else:
            dist.init_process_group(backend, rank=rank, world_size=world, device_id=device_id)
    except Exception as e:  # noqa: BLE001
        q.put(("init-failed", rank, repr(e)))
        raise
