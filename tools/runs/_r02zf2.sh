set -u
for w in resnet50 alexnet_bn; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_zff32.so --workload $w --reps 3 2>&1 | tail -2
done
