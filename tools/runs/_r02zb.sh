set -u
LARS_B200_LIB=liblars_b200_w16.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size or golden or sweep_layouts or carry" 2>&1 | tail -2
for w in resnet50 alexnet_bn sweep:16e6:100; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_w16.so --workload $w --reps 3 2>&1 | tail -2
done
for lib in liblars_b200.so liblars_b200_w16.so; do
  echo "== shard $lib"; LARS_B200_LIB=$lib timeout 600 python tools/shard_time.py --workloads resnet50,sweep:1e6:50 --worlds 1,4,8 2>&1 | tail -1
done
