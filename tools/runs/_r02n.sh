set -u
out=gpurun_out/r02n
mkdir -p $out
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "bench n$n rc=$?"
  cut -c 1-300 $out/bench_n$n.json; grep -i -A5 "double free\|Traceback\|Error" $out/bench_n$n.err | head -20
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --impl reference --steps 5 --warmup 1 > $out/bench_ref_n$n.json 2> $out/bench_ref_n$n.err; echo "ref n$n rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus 4 --backend nccl --train-steps 0 > $out/bench_nccl_n4.json 2> $out/bench_nccl_n4.err; echo "nccl n4 rc=$?"
