set -u
out=gpurun_out/r02final4b
mkdir -p $out
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench n1 rc=$?"
for k in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 --master-port 2965$k bench.py --gpus $k > $out/bench_n$k.json 2> $out/bench_n$k.err; echo "bench n$k rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "overlap or desync or (p2p-stream and sharded_step and resnet50) or (nccl and sharded_step and alexnet)" > $out/pytest_dist_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_dist_subset.log
