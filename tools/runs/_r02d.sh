set -u
out=gpurun_out/r02d
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests/test_gpu_dist.py -q -rs --durations=12 > $out/pytest_gpu_dist_n$n.log 2>&1; echo "pytest rc=$?"
tail -30 $out/pytest_gpu_dist_n$n.log
