set -u
out=gpurun_out/r02f
mkdir -p $out
for w in resnet50 alexnet_bn; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_f64w.so liblars_b200_f32.so --workload $w --reps 3 2>&1 | tail -3
done
for lib in liblars_b200.so liblars_b200_f64w.so liblars_b200_f32.so; do
  echo "== shard $lib"
  LARS_B200_LIB=$lib timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn --worlds 1,4,8 2>&1 | tail -1
done
