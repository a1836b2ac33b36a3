for rep in 1 2; do
  for lib in liblars_b200.so liblars_b200_ku1.so liblars_b200_ku3.so; do
    LARS_B200_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2978$rep bench.py --gpus 4 --train-steps 0 --steps 50 --e2e-steps 2 --no-traffic > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$lib', d['ms_per_step'])" || tail -3 /tmp/b.err
  done
done
