set -u
LARS_DEBUG_OCC=1 python -c "
import torch
from paper_1709_05011_b200 import layouts
from paper_1709_05011_b200.flat import FlatParamSet
f=FlatParamSet(layouts.get('resnet50'),'cuda')
p,_=f.engine().plan(frozenset({'bias','norm-scale','norm-shift'}))
print('grid', p.info.grid, 'smem', p.info.smem_bytes)
"
