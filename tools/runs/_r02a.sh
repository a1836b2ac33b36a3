set -u
out=gpurun_out/r02a
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
cat $out/bench_n1.json
timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn,sweep:1e6:50,sweep:16e6:100 > $out/shard_time.jsonl 2> $out/shard_time.err; echo "shard rc=$?"
cat $out/shard_time.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20
