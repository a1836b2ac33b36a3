set -u
run() {
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 4 --backend nccl --train-steps 0 --steps 30 --e2e-steps 2 > /tmp/n.json 2>/tmp/n.err
  python -c "import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('$*', d['ms_per_step'], d['phases_us'], d.get('busbw_gbs'))" || (echo "$* failed"; tail -3 /tmp/n.err)
}
run NCCL_DEBUG=WARN
run NCCL_NVLS_ENABLE=0
run NCCL_ALGO=Ring NCCL_PROTO=Simple
run NCCL_ALGO=NVLS
run NCCL_MIN_NCHANNELS=32
run NCCL_MIN_NCHANNELS=32 NCCL_NVLS_ENABLE=0
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 4 --backend nccl --train-steps 0 --steps 3 --warmup 3 --e2e-steps 1 2>&1 | grep -iE "nvls|algo|channel|ring" | head -15
