set -u
out=gpurun_out/r02final4
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=8 > $out/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"
