LARS_B200_LIB=liblars_b200_ca2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or full_size or carry or sweep or grid" 2>&1 | tail -1
for w in resnet50 alexnet_bn sweep:16e6:100 sweep:1e6:50; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_ca2.so --workload $w --reps 3 2>&1 | tail -2
done
