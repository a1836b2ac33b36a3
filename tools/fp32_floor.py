"""fp32-state error floor of the 100-step ResNet-50 trajectory test
(tests/test_gpu_trajectory.py): one layer stepped 100 times with fp32 w / m
in numpy (the kernel's arithmetic) vs the fp64 oracle.  CPU only."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tests"), ROOT]
import numpy as np, gen
from helpers import rolled_grads
from paper_1709_05011_b200 import layouts
from oracle import lars_oracle as orc
L=layouts.get('resnet50'); idx=[i for i,(n,_,_) in enumerate(L) if n=='layer3.0.downsample.0.weight'][0]
ins=gen.group_inputs(L,17)
base=gen.step_grads(L,17,0,g_scale=1e-3)
w,g,m=ins[idx]; b=[base[idx]]
# rolled_grads uses group index i in the roll offset -> emulate with i=idx
def rg(t):
    s=np.float32((-1.0)**t*2.0**((t%3)-1)); return (np.roll(base[idx].reshape(-1),7919*t+13*idx)*s)
class H: pass
hp=H(); hp.base_lr=25.6; hp.warmup_epochs=5; hp.poly_power=2.0
w64=w.reshape(-1).astype(np.float64); m64=m.reshape(-1).astype(np.float64)
w32=w.reshape(-1).copy(); m32=m.reshape(-1).copy()
for t in range(100):
    it=150+t; lr=orc.scheduled_lr(hp,it,3515,39)
    gt=rg(t)
    g64=gt.astype(np.float64)
    lam=orc.lars_local_lr(w64,g64,5e-4,1e-3)
    s=g64+5e-4*w64; m64=m64*0.9+(lam*lr)*s; w64=w64-m64
    lam32=orc.lars_local_lr(w32.astype(np.float64),gt.astype(np.float64),5e-4,1e-3)
    k=np.float32(lam32*lr)
    sg=np.float32(5e-4)*w32+gt  # approx fma
    m32=(np.float32(0.9)*m32+k*sg).astype(np.float32); w32=(w32-m32).astype(np.float32)
rms=np.sqrt(np.mean(w64**2)); err=np.abs(w32-w64)
print('rms',rms,'max err',err.max(),'max err/rms',err.max()/rms, 'median err/rms', np.median(err)/rms)
tol=1e-4*np.abs(w64)+1e-6*rms
print('viol',(err>tol).sum(), 'worst ratio',(err/tol).max())
