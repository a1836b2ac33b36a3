set -u
out=gpurun_out/r02m
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
for i in 1 2; do
PYTHONFAULTHANDLER=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus $n --train-steps 2 > $out/bench_n${n}_$i.json 2> $out/bench_n${n}_$i.err; echo "bench rc=$?"
cat $out/bench_n${n}_$i.json | cut -c 1-400; grep -v "Warn" $out/bench_n${n}_$i.err | grep -i -B3 -A25 "fatal\|double free\|Traceback" | head -60
done
