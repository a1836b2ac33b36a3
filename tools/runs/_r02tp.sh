for w in resnet50 alexnet_bn sweep:16e6:100 sweep:1e6:50; do
  echo "== ab $w"; timeout 900 python tools/ab_time.py liblars_b200.so liblars_b200_t1.so liblars_b200_t2.so liblars_b200_t3.so liblars_b200_t4.so liblars_b200_t5.so --workload $w --reps 2 2>&1 | tail -6
done
