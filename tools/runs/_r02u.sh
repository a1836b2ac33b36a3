set -u
out=gpurun_out/r02u
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
timeout 2700 python -m pytest tests/test_gpu_dist.py -q -rs --durations=10 > $out/pytest_gpu_dist_n$n.log 2>&1; echo "pytest rc=$?"
tail -22 $out/pytest_gpu_dist_n$n.log
