set -u
out=gpurun_out/r02e
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lo tools/launch_overhead.cu && timeout 120 /tmp/lo > $out/launch_overhead.txt 2>&1; cat $out/launch_overhead.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py tests/test_c_abi.py -q -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for w in resnet50 alexnet_bn sweep:1e6:50 sweep:16e6:100; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_f32.so --workload $w --reps 3 2>&1 | tail -3
done
timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn,sweep:1e6:50 > $out/shard_time.jsonl 2>&1; tail -1 $out/shard_time.jsonl
export LARS_B200_LIB=liblars_b200_trace.so
for spec in "sweep:1e6:50 1 0" "resnet50 8 0" "resnet50 1 0"; do
  set -- $spec
  echo "== trace $1 world $2 rank $3"
  timeout 300 python tools/trace_step.py --workload $1 --world $2 --rank $3 --steps 6 2>&1 | head -14
done
