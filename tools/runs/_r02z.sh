set -u
out=gpurun_out/r02z
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
{
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/soak.py --steps 1500 --workload resnet50
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/soak.py --steps 500 --workload alexnet_bn
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/soak.py --steps 1000 --workload sweep:2e6:1500
for be in p2p p2p-stream nccl; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960${#be} tools/soak.py --steps 600 --workload resnet50 --backend $be 2>&1 | grep soak
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 tools/soak.py --steps 1000 --workload mlp --backend p2p 2>&1 | grep soak
} > $out/soak.txt 2>&1
cat $out/soak.txt
