set -u
out=gpurun_out/r02w
mkdir -p $out
timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn,sweep:1e6:50,sweep:16e6:100 --worlds 1,2,4,8 > $out/shard_time.jsonl 2>&1; tail -1 $out/shard_time.jsonl
for w in sweep:1e6:50 sweep:16e6:100 sweep:256e6:200 sweep:1e9:300; do
  f=$out/$(echo $w | tr ':' '_')_n1.json
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --train-steps 0 --e2e-steps 2 --host-e2e-steps 0 --no-cpu-baseline > $f 2>/dev/null
  echo "$w rc=$? $(cut -c 1-200 $f)"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sweep or grid or carry or full_size" 2>&1 | tail -2
