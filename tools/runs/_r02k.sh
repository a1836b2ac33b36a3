set -u
for w in resnet50 alexnet_bn sweep:16e6:100; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_c2.so liblars_b200_c4.so liblars_b200_c8.so --workload $w --reps 3 2>&1 | tail -4
done
for lib in liblars_b200.so liblars_b200_c4.so; do
  echo "== shard $lib"
  LARS_B200_LIB=$lib timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn --worlds 1,4,8 2>&1 | tail -1
done
