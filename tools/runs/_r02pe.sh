set -u
mkdir -p gpurun_out/r02pe
LARS_B200_LIB=liblars_b200_pe.so timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x -k "(p2p and not stream and not trajectory and not overlap) or (trajectory and p2p-2-resnet50) or (trajectory and p2p-4-resnet50)" > gpurun_out/r02pe/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02pe/pytest.log
for rep in 1 2; do
for k in 4 2; do
  for lib in liblars_b200.so liblars_b200_pe.so; do
    LARS_B200_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 --master-port 2977$k bench.py --gpus $k --train-steps 0 --steps 50 --e2e-steps 2 --no-traffic > /tmp/b.json 2>/tmp/b.err
    python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$lib', 'n$k', d['ms_per_step'], d['scaling_defs']['step_roofline_eff'])" || tail -3 /tmp/b.err
  done
done
done
timeout 600 python tools/ab_time.py liblars_b200.so liblars_b200_pe.so --workload resnet50 --reps 2 2>&1 | tail -2
