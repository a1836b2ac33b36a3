set -u
n=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -k "p2p-stream and not 8" > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -3 /tmp/pt.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29590 bench.py --gpus $n --backend p2p-stream --train-steps 0 --steps 30 > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('stream',d['ms_per_step'],d['roofline']['kernel_us'],d['scaling_defs']['step_roofline_eff'])" || tail -3 /tmp/b.err
LARS_B200_LIB=liblars_b200_trace.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29593 tools/trace_stream.py --workload resnet50 2>&1 | grep -v Warn | tail -3
