set -u
out=gpurun_out/r02final4c
mkdir -p $out
timeout 2700 python -m pytest tests/test_gpu_dist.py -q -rs --durations=6 > $out/pytest_gpu_dist_n4.log 2>&1; echo "pytest rc=$?"
tail -6 $out/pytest_gpu_dist_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29670 bench.py --gpus 4 --backend nccl --train-steps 0 > $out/bench_nccl_n4.json 2> $out/bench_nccl_n4.err; echo "nccl rc=$?"
for k in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 --master-port 2966$k bench.py --gpus $k --impl reference --steps 5 --warmup 1 > $out/bench_ref_n$k.json 2> $out/bench_ref_n$k.err; echo "ref n$k rc=$?"
done
