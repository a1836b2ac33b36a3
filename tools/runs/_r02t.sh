set -u
out=gpurun_out/r02t
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=12 > $out/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"
tail -20 $out/pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $out/smoke.log
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
cut -c 1-600 $out/bench_n1.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"
timeout 600 python bench.py --workload alexnet_bn --train-steps 0 > $out/bench_abn_n1.json 2> $out/bench_abn_n1.err; echo "abn rc=$?"
cut -c 1-400 $out/bench_abn_n1.json
