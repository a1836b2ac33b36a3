set -u
out=gpurun_out/r02h
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests/test_gpu_dist.py -q -rs --durations=8 > $out/pytest_gpu_dist_n$n.log 2>&1; echo "pytest rc=$?"
tail -25 $out/pytest_gpu_dist_n$n.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 50 --warmup 5 > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "bench rc=$?"
cat $out/bench_n$n.json; tail -5 $out/bench_n$n.err
