set -u
for k in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 --master-port 2967$k bench.py --gpus $k --train-steps 0 > /tmp/b$k.json 2> /tmp/b$k.err; echo "bench n$k rc=$?"
  python -c "import json;d=json.loads(open('/tmp/b$k.json').read().strip().splitlines()[-1]);print($k,d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs'])" || tail -5 /tmp/b$k.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29679 bench.py --gpus 4 --backend nccl --train-steps 0 > /tmp/bn.json 2> /tmp/bn.err; echo "nccl rc=$?"
python -c "import json;d=json.loads(open('/tmp/bn.json').read().strip().splitlines()[-1]);print('nccl',d['ms_per_step'],d['phases_us'],d['scaling_defs']['step_roofline_eff'])" || tail -5 /tmp/bn.err
