#!/bin/bash
# One-GPU evidence run (gpurun): GPU tests, smoke, the default bench line,
# the ncu launch list of a short bench, and one `ncu --set full` capture of
# the step kernel per workload.  Outputs under gpurun_out/evidence/.
set -u
out=gpurun_out/evidence
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
cat $out/bench_n1.json
# the ncu passes only after the commands above exited 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_bench_n1.csv \
  python bench.py --steps 5 --warmup 3 --train-steps 0 --no-cpu-baseline --e2e-steps 2 \
  > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for w in resnet50 alexnet_bn; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:lars_step_kernel \
    --launch-skip 2 --launch-count 1 -o $out/lars_step_$w -f \
    python tools/profile_step.py --workload $w --steps 3 > $out/ncu_$w.log 2>&1
  echo "ncu $w rc=$?"
done
