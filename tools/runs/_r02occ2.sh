set -u
LARS_DEBUG_OCC=1 python -c "
from paper_1709_05011_b200 import layouts
from paper_1709_05011_b200.flat import FlatParamSet
f=FlatParamSet(layouts.get('resnet50'),'cuda')
p,_=f.engine().plan(frozenset({'bias','norm-scale','norm-shift'}))
print('grid', p.info.grid, 'smem', p.info.smem_bytes)
" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_size or golden or full_size" 2>&1 | tail -1
for w in resnet50 sweep:1e6:50; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200_head.so liblars_b200.so --workload $w --reps 3 2>&1 | tail -2
done
