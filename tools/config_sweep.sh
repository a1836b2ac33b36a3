#!/bin/bash
# BASELINE configs 2/3/5 through bench.py on 1, 2 and 4 GPUs (gpurun --gpus 4):
# AlexNet-BN and the standalone sweep (1M..1B parameters).  One JSON line per
# run under gpurun_out/sweep/; summarise with tools/config_sweep_table.py.
set -u
out=gpurun_out/sweep
mkdir -p $out
port=29600
for w in alexnet_bn sweep:1e6:50 sweep:16e6:100 sweep:256e6:200 sweep:1e9:300; do
  for n in 1 2 4; do
    port=$((port + 1))
    f=$out/$(echo $w | tr ':' '_')_n$n.json
    if [ $n -eq 1 ]; then
      timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --train-steps 0 \
        --no-cpu-baseline --e2e-steps 2 2>/dev/null | grep metric > $f
    else
      timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
        bench.py --gpus $n --workload $w --steps 20 --warmup 3 --train-steps 0 --e2e-steps 2 \
        2>/dev/null | grep metric > $f
    fi
    echo "$w n=$n rc=$? $(head -c 160 $f)"
  done
done
