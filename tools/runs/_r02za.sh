set -u
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29620 tools/soak.py --steps 600 --workload resnet50 --backend p2p-stream > /tmp/s.out 2>&1; echo "rc=$?"
grep -v Warn /tmp/s.out | tail -30
