import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
from paper_1709_05011_b200 import hostset, layouts, optim
layout = layouts.get("resnet50")
ref = bench.stock_reference()
params = bench._stock_paramset(ref, layout) if ref is not None else bench._oracle_groups(layout)
hp = optim.HyperParams(**bench._recipe_kw())
for _ in range(3):
    optim.apply_update(params, hp, 0.1, iteration=0)
mirror, groups = hostset.mirror_for(params)
# instrument: wrap _load_part/_store_part with events
ev = []
orig_load, orig_store = mirror._load_part, mirror._store_part
def load(groups, part, live):
    a = torch.cuda.Event(enable_timing=True); a.record()
    orig_load(groups, part, live)
    b = torch.cuda.Event(enable_timing=True); b.record()
    ev.append(("load", part.g0, a, b, time.perf_counter()))
def store(groups, part, upto=None):
    a = torch.cuda.Event(enable_timing=True); a.record()
    r = orig_store(groups, part, upto)
    b = torch.cuda.Event(enable_timing=True); b.record()
    ev.append(("store", part.g0, a, b, time.perf_counter()))
    return r
mirror._load_part, mirror._store_part = load, store
t0 = time.perf_counter()
z = torch.cuda.Event(enable_timing=True); z.record()
optim.apply_update(params, hp, 0.1, iteration=0)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"wall {1e3*(t1-t0):.2f} ms, parts {len(mirror.parts)}")
for name, g0, a, b, th in ev:
    print(f"{name:5s} part@{g0:3d}: gpu {z.elapsed_time(a):7.2f} -> {z.elapsed_time(b):7.2f} ms   host enqueue done at {1e3*(th-t0):7.2f} ms")
