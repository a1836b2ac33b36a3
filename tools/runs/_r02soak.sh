for spec in "4 resnet50 600" "4 alexnet_bn 300" "4 sweep:2e6:1500 400" "2 resnet50 600"; do
  set -- $spec
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2990$1 tools/soak.py --workload $2 --steps $3 --backend p2p 2>/dev/null | tail -1
done
