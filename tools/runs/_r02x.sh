set -u
n=$(nvidia-smi -L | wc -l)
for lib in liblars_b200.so liblars_b200_aw7.so liblars_b200_aw8.so; do
  LARS_B200_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29590 bench.py --gpus $n --backend p2p-stream --train-steps 0 --steps 30 --e2e-steps 2 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$lib stream',d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs']['step_roofline_eff'])" || tail -3 /tmp/b.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $n --backend p2p --train-steps 0 --steps 30 --e2e-steps 2 > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('p2p',d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs']['step_roofline_eff'])"
