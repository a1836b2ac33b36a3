"""A/B timing of LARS step library variants in ONE process-per-variant run.

    python tools/ab_time.py libA.so libB.so ... [--workload resnet50] [--reps 3]

Each variant runs in a subprocess (LARS_B200_LIB=<name>), timing 30 eager
fused steps with CUDA events (L2 flushed before each), and the median is
printed; variants are interleaved `--reps` times to average out drift.
"""
import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, statistics
sys.path.insert(0, %r)
import torch
if os.environ.get("LARS_L2_PERSIST"):
    from cuda.bindings import runtime as rt
    torch.cuda.init(); torch.zeros(1, device="cuda")
    err, mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
    want = min(mx, int(float(os.environ["LARS_L2_PERSIST"]) * (1 << 20)))
    print("persist max", mx, "set", want, rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, want), file=sys.stderr)
from paper_1709_05011_b200 import layouts, optim
from paper_1709_05011_b200.cluster import DataParallelLars
from paper_1709_05011_b200.flat import FlatParamSet
dev = torch.device("cuda:0")
layout = layouts.get(%r)
params = FlatParamSet(layout, dev)
g = torch.Generator(device=dev); g.manual_seed(1)
if os.environ.get("AB_BENCH_DATA"):  # bench.py's inputs
    for grp in params:
        if grp.category == "norm-scale":
            grp.param.fill_(1.0)
        elif grp.category == "weight":
            grp.param.uniform_(-0.05, 0.05, generator=g)
        grp.grad.normal_(0.0, 32.768, generator=g)
else:
    for grp in params:
        grp.param.uniform_(-0.05, 0.05, generator=g)
        grp.grad.normal_(0, 1.0, generator=g)
hp = optim.HyperParams(base_lr=25.6, epochs=90, batch_size=32768, warmup_epochs=5, lars_enabled=True)
st = optim.ScheduleState(3515, 39)
dp = DataParallelLars(params)
flush = torch.empty(1 << 28, dtype=torch.float32, device=dev)
clean = torch.ones(1 << 26, dtype=torch.float32, device=dev)
ts = []
for i in range(40):
    flush.zero_(); clean.sum()
    t = []
    dp.step(hp, st, grad_scale=1.0 / 32768, timers=t)
    if i >= 10:
        ts.append(t)
torch.cuda.synchronize()
ms = [t[0][1].elapsed_time(t[1][1]) for t in ts]
print(json.dumps(statistics.median([x * 1e3 for x in ms])))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "resnet50"
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    libs = [a for a in args if a.endswith(".so")]
    persists = os.environ.get("AB_PERSIST", "").split(",") if os.environ.get("AB_PERSIST") else [""]
    libs = [(l, p) for l in libs for p in persists]
    res = {l: [] for l in libs}
    for _ in range(reps):
        for lib, pers in libs:
            env = dict(os.environ, LARS_B200_LIB=lib)
            if pers:
                env["LARS_L2_PERSIST"] = pers
            out = subprocess.run([sys.executable, "-c", CHILD % (HERE, wl)], env=env,
                                 capture_output=True, text=True)
            try:
                res[(lib, pers)].append(json.loads(out.stdout.strip().splitlines()[-1]))
            except Exception:
                print(lib, "failed:", out.stderr[-2000:])
            if pers and res[(lib, pers)] and len(res[(lib, pers)]) == 1:
                print("  ", out.stderr.strip().splitlines()[-1][:200] if out.stderr.strip() else "")
    for (lib, pers), v in res.items():
        if v:
            print(f"{lib:32s} persist={pers or '-':6s} us: " + " ".join(f"{x:7.2f}" for x in v) +
                  f"   median {statistics.median(v):7.2f}")


if __name__ == "__main__":
    main()
