"""Generate tests/golden/lars_golden.npz + manifest.json by running the
REFERENCE implementation itself (batchlab, imported read-only from
/root/reference/pkg/src) on the inputs of tests/golden/gen.py.

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Every case records the reference's outputs in fp64: final weights and
momentum (flat, group order), the last step's lambdas and learning rate.
The calls used are the reference's own: optim.sgd_step / apply_update
(optim.py:117-142), optim.scheduled_lr (:76-95), cluster.all_reduce
(cluster.py:124-137) followed by `/ b` (cluster.py:147-148).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("BATCHLAB_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from batchlab import cluster, nn, optim  # noqa: E402  (the reference)
from batchlab.errors import DivergenceError  # noqa: E402

import gen  # noqa: E402
from paper_1709_05011_b200 import layouts  # noqa: E402  (shape tables only)

LAYOUTS = {"ragged": gen.RAGGED, "mlp": layouts.mlp(), "lenet5": layouts.lenet5()}

HP = {
    # config 1 recipe: lars on, warmup, poly 2
    "lars_warm": dict(base_lr=0.32, epochs=10, batch_size=512, momentum=0.9,
                      weight_decay=5e-4, poly_power=2.0, warmup_epochs=2,
                      lars_enabled=True, lars_trust=1e-3),
    "plain": dict(base_lr=0.1, epochs=10, batch_size=32, momentum=0.9,
                  weight_decay=5e-4, poly_power=2.0, warmup_epochs=0, lars_enabled=False),
    "lars_nowd": dict(base_lr=0.05, epochs=10, batch_size=32, momentum=0.0,
                      weight_decay=0.0, poly_power=2.0, warmup_epochs=0,
                      lars_enabled=True, lars_trust=1e-2),
    "lars_sqrt": dict(base_lr=2.0, epochs=10, batch_size=64, momentum=0.9,
                      weight_decay=1e-4, poly_power=0.5, warmup_epochs=0,
                      lars_enabled=True, lars_trust=2e-3),
    "lars_big": dict(base_lr=25.6, epochs=10, batch_size=32768, momentum=0.9,
                     weight_decay=5e-4, poly_power=2.0, warmup_epochs=5,
                     lars_enabled=True, lars_trust=1e-3),
}

CASES = [
    # name, layout, hp, seed, (max_iters, ipe, iteration), steps, extra
    ("ragged_lars_warm", "ragged", "lars_warm", 1, (100, 10, 0), 1, {}),
    ("ragged_lars_mid", "ragged", "lars_warm", 2, (100, 10, 37), 1, {}),
    ("ragged_plain", "ragged", "plain", 3, (100, 10, 5), 1, {}),
    ("ragged_nowd_zero", "ragged", "lars_nowd", 4, (100, 10, 0), 1,
     {"zero_w": ["zero.weight"], "zero_g": ["nograd.weight"]}),
    ("ragged_sqrt_end", "ragged", "lars_sqrt", 5, (50, 5, 50), 1, {}),
    ("ragged_big_lr", "ragged", "lars_big", 6, (3906, 39, 100), 1, {}),
    ("lenet5_lars", "lenet5", "lars_warm", 7, (100, 10, 3), 1, {}),
    ("mlp_lars_1", "mlp", "lars_warm", 8, (200, 10, 0), 1, {}),
    ("mlp_lars_100", "mlp", "lars_warm", 8, (200, 10, 0), 100, {}),
    ("ragged_traj_100", "ragged", "lars_sqrt", 9, (120, 4, 0), 100, {}),
    ("ragged_explicit_lr", "ragged", "lars_warm", 10, (100, 10, 0), 1,
     {"explicit_lr": 0.7, "iteration": 12}),
    ("ragged_dp4", "ragged", "lars_warm", 11, (100, 10, 30), 1, {"dp": 4, "local_batch": 128}),
    ("mlp_dp8", "mlp", "lars_warm", 12, (100, 10, 25), 1, {"dp": 8, "local_batch": 64}),
]


def make_hp(name):
    d = dict(HP[name])
    return optim.HyperParams(**d)


def build_paramset(layout, seed, extra):
    groups = []
    ins = gen.group_inputs(layout, seed, zero_w=tuple(extra.get("zero_w", ())),
                           zero_g=tuple(extra.get("zero_g", ())))
    for (name, shape, cat), (w, g, m) in zip(layout, ins):
        groups.append(nn.ParamGroup(name, w.astype(np.float64), g.astype(np.float64),
                                    m.astype(np.float64), cat))
    return nn.ParamSet(groups)


def run_case(name, lay, hpn, seed, stv, steps, extra):
    layout = LAYOUTS[lay]
    hp = make_hp(hpn)
    ps = build_paramset(layout, seed, extra)
    st = optim.ScheduleState(max_iterations=stv[0], iterations_per_epoch=stv[1], iteration=stv[2])
    lams, lr = None, None
    for t in range(steps):
        if t > 0:
            for grp, g in zip(ps, gen.step_grads(layout, seed, t)):
                np.copyto(grp.grad, g.astype(np.float64))
        if "dp" in extra:
            P, lb = extra["dp"], extra["local_batch"]
            # per-worker sum-convention gradients (cluster.local_gradients)
            sets = []
            for r in range(P):
                gs = gen.step_grads(layout, seed * 31 + r, 0, g_scale=1e-3 * lb)
                sets.append({grp.name: g.astype(np.float64) for grp, g in zip(ps, gs)})
            summed = cluster.all_reduce(sets)                       # cluster.py:146
            b = P * lb
            mean = {k: v / b for k, v in summed.items()}            # cluster.py:147-148
            lr = optim.scheduled_lr(hp, st)                         # cluster.py:149
            ps.set_grads(mean)                                      # cluster.py:152
            lams = optim.apply_update(ps, hp, lr, iteration=st.iteration)  # :153
            st.iteration += 1                                       # :154
        elif "explicit_lr" in extra:
            lr = extra["explicit_lr"]
            lams = optim.apply_update(ps, hp, lr, iteration=extra["iteration"])
        else:
            lr = optim.scheduled_lr(hp, st)
            lams = optim.sgd_step(ps, hp, st)
    w = np.concatenate([g.param.reshape(-1) for g in ps])
    m = np.concatenate([g.momentum_buf.reshape(-1) for g in ps])
    lam = np.array([lams[g.name] for g in ps], dtype=np.float64)
    return w, m, lam, float(lr), st.iteration


def divergence_case():
    layout = gen.RAGGED
    ps = build_paramset(layout, 13, {})
    ps["b.weight"].grad[:] = np.inf
    hp = make_hp("plain")
    try:
        optim.apply_update(ps, hp, lr=1.0, iteration=42)
    except DivergenceError as e:
        return {"iteration": e.iteration, "message": str(e)}
    raise AssertionError("reference did not diverge")


def schedule_case():
    rows = []
    for hpn, (mx, ipe) in [("lars_warm", (100, 10)), ("lars_sqrt", (50, 5)),
                           ("lars_big", (3906, 39)), ("plain", (14062, 281))]:
        hp = make_hp(hpn)
        for it in sorted({0, 1, ipe - 1, ipe, 2 * ipe - 1, 2 * ipe, mx // 2, mx - 1, mx}):
            st = optim.ScheduleState(max_iterations=mx, iterations_per_epoch=ipe, iteration=it)
            rows.append([hpn, mx, ipe, it, optim.scheduled_lr(hp, st)])
    return rows


def main():
    arrays = {}
    manifest = {"hp": HP, "cases": [], "reference": REF}
    for name, lay, hpn, seed, stv, steps, extra in CASES:
        w, m, lam, lr, it_after = run_case(name, lay, hpn, seed, stv, steps, extra)
        arrays[f"{name}/w"] = w
        arrays[f"{name}/m"] = m
        arrays[f"{name}/lambda"] = lam
        manifest["cases"].append(dict(name=name, layout=lay, hp=hpn, seed=seed,
                                      max_iters=stv[0], ipe=stv[1], iteration=stv[2],
                                      steps=steps, extra=extra, lr=lr,
                                      iteration_after=it_after))
    manifest["divergence"] = divergence_case()
    manifest["schedule"] = schedule_case()
    np.savez_compressed(os.path.join(HERE, "lars_golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print(f"{len(CASES)} cases written")


if __name__ == "__main__":
    main()
