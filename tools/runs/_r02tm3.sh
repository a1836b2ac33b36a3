set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py tests/test_c_abi.py tests/test_telemetry.py -q -x -m gpu 2>&1 | tail -3
for w in resnet50 alexnet_bn sweep:16e6:100 sweep:1e6:50; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200_head.so liblars_b200_notmem.so liblars_b200.so --workload $w --reps 3 2>&1 | tail -3
done
