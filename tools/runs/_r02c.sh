set -u
out=gpurun_out/r02c
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x -rs --durations=10 > $out/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"
tail -16 $out/pytest_gpu_n1.log
export LARS_B200_LIB=liblars_b200_trace.so
for spec in "sweep:1e6:50 1 0" "resnet50 8 0" "resnet50 8 5" "alexnet_bn 8 0" "resnet50 1 0"; do
  set -- $spec
  echo "== trace $1 world $2 rank $3"
  timeout 300 python tools/trace_step.py --workload $1 --world $2 --rank $3 --steps 6 2>&1 | head -14
done
