set -u
out=gpurun_out/r02p
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "p2p-stream and not 8" -rs > $out/pytest_stream_n$n.log 2>&1; echo "pytest rc=$?"
tail -30 $out/pytest_stream_n$n.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29580 bench.py --gpus $n --backend p2p-stream --train-steps 0 > $out/bench_stream_n$n.json 2> $out/bench_stream_n$n.err; echo "bench rc=$?"
cut -c 1-1500 $out/bench_stream_n$n.json; grep -i "error\|Traceback" $out/bench_stream_n$n.err | head
