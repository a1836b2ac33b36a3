set -u
out=gpurun_out/r02b
mkdir -p $out
nvidia-smi --query-gpu=name --format=csv,noheader | head -8
timeout 1500 python -m pytest tests -m gpu -q -x -rs --durations=15 > $out/pytest_gpu_n${NGPU:-1}.log 2>&1; echo "pytest rc=$?"
tail -30 $out/pytest_gpu_n${NGPU:-1}.log
