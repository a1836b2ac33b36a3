set -u
out=gpurun_out/r02j
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "bench rc=$?"
cat $out/bench_n$n.json; grep -v Warn $out/bench_n$n.err | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --impl reference --steps 5 --warmup 1 > $out/bench_ref_n$n.json 2> $out/bench_ref_n$n.err; echo "ref rc=$?"; cat $out/bench_ref_n$n.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus $n --backend nccl --train-steps 0 > $out/bench_nccl_n$n.json 2> $out/bench_nccl_n$n.err; echo "bench nccl rc=$?"; cat $out/bench_nccl_n$n.json
