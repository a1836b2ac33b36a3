set -u
out=gpurun_out/r02l
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
python tools/nvlink_counters.py --index 0 > $out/nvml_before.json 2>&1; cat $out/nvml_before.json
nvidia-smi nvlink -gt d -i 0 > $out/smi_before.txt 2>&1; head -8 $out/smi_before.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29540 tools/nvls_bw.py > $out/nvls_bw.txt 2>&1; tail -4 $out/nvls_bw.txt
python tools/nvlink_counters.py --index 0 > $out/nvml_after.json 2>&1; cat $out/nvml_after.json
nvidia-smi nvlink -gt d -i 0 > $out/smi_after.txt 2>&1; head -8 $out/smi_after.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "bench rc=$?"
cat $out/bench_n$n.json
