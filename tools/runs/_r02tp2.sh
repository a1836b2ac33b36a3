LARS_B200_LIB=liblars_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py -q -x -k "full_size or carry or sweep or grid or hundred" 2>&1 | tail -1
for w in alexnet_bn sweep:64e6:100 resnet50 sweep:16e6:100; do
  echo "== ab $w"; timeout 900 python tools/ab_time.py liblars_b200_base.so liblars_b200.so --workload $w --reps 3 2>&1 | tail -2
done
