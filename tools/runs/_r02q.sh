set -u
n=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -k "p2p-stream and not 8 and not trajectory" > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -2 /tmp/pt.log
for lib in liblars_b200.so liblars_b200_aw2.so liblars_b200_aw6.so; do
  for be in p2p-stream; do
    LARS_B200_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29590 bench.py --gpus $n --backend $be --train-steps 0 --steps 30 > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$lib','$be',d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs']['step_roofline_eff'])" || tail -3 /tmp/b.err
  done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $n --backend p2p --train-steps 0 --steps 30 > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('p2p',d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs']['step_roofline_eff'])"
