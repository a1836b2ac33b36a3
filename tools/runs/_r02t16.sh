set -u
LARS_TMEM_PLAN=1 LARS_B200_LIB=liblars_b200_t16.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py -q -x -k "golden or full_size or carry or sweep or hundred" 2>&1 | tail -2
for w in resnet50 alexnet_bn sweep:16e6:100; do
  echo "== ab $w"; LARS_TMEM_PLAN=1 timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_w16n.so liblars_b200_t16.so --workload $w --reps 3 2>&1 | tail -3
done
