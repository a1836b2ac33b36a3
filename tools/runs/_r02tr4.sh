set -u
n=$(nvidia-smi -L | wc -l)
LARS_B200_LIB=liblars_b200_trace.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29694 tools/trace_nvls.py --workload resnet50 --steps 6 2>&1 | grep -v Warn | tail -8
