set -u
out=gpurun_out/r02final2
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=8 > $out/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"
tail -14 $out/pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
cut -c 1-300 $out/bench_n1.json
timeout 600 python bench.py --impl reference > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_n1.csv \
  python bench.py --steps 5 --warmup 3 --train-steps 0 --no-cpu-baseline --e2e-steps 2 --host-e2e-steps 2 --no-traffic > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lars_step_kernel \
    --launch-skip 3 --launch-count 1 -o $out/lars_step_resnet50 -f \
    python tools/profile_step.py --workload resnet50 --steps 5 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
