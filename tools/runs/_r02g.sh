set -u
for w in resnet50 alexnet_bn; do
  for cfg in "" "LARS_POL_B=0" "LARS_KEEP_MB=40 LARS_POL_B=0" "LARS_KEEP_MB=60 LARS_POL_B=0" "LARS_KEEP_MB=80 LARS_POL_B=0" "LARS_KEEP_MB=60" "LARS_KEEP_MB=80"; do
    echo "== $w [$cfg]"; env $cfg timeout 300 python tools/ab_time.py liblars_b200.so --workload $w --reps 2 2>&1 | tail -1
  done
done
