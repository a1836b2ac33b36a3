set -u
for w in resnet50 alexnet_bn sweep:16e6:100; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_a20.so liblars_b200_a24.so --workload $w --reps 3 2>&1 | tail -3
done
for g in 148 222 296; do
  echo "== shard grid $g"
  timeout 600 python tools/shard_time.py --workloads resnet50,sweep:1e6:50 --worlds 4,8 --grid $g 2>&1 | tail -1
done
