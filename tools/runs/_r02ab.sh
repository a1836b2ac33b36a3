set -u
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py tests/test_c_abi.py -q -x -k "not hundred" 2>&1 | tail -2
for w in resnet50 alexnet_bn sweep:16e6:100 sweep:1e6:50; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200_prev.so liblars_b200.so --workload $w --reps 3 2>&1 | tail -2
done
for lib in liblars_b200_prev.so liblars_b200.so; do
  echo "== shard $lib"; LARS_B200_LIB=$lib timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn --worlds 1,4,8 2>&1 | tail -1
done
