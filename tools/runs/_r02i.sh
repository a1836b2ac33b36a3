set -u
out=gpurun_out/r02i
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cvt tools/cvt_throughput.cu && /tmp/cvt > $out/cvt_throughput.txt 2>&1; cat $out/cvt_throughput.txt
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
cat $out/bench_n1.json; tail -3 $out/bench_n1.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 2 > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"; cat $out/bench_ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_n1.csv \
  python bench.py --steps 5 --warmup 3 --train-steps 0 --no-cpu-baseline --e2e-steps 2 --host-e2e-steps 2 --no-traffic > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for spec in "resnet50 1 0" "alexnet_bn 1 0" "resnet50 8 0"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:lars_step_kernel \
    --launch-skip 3 --launch-count 1 -o $out/lars_step_$1_w$2 -f \
    python tools/profile_step.py --workload $1 --world $2 --rank $3 --steps 5 > $out/ncu_$1_w$2.log 2>&1
  echo "ncu $1 w$2 rc=$?"
done
