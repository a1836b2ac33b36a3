for w in resnet50 alexnet_bn; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200_old.so liblars_b200.so --workload $w --reps 3 2>&1 | tail -2
done
mkdir -p gpurun_out/r02ab2
timeout 900 python bench.py > gpurun_out/r02ab2/bench_n1.json 2> gpurun_out/r02ab2/bench_n1.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02ab2/bench_n1.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_us'], d['e2e']['ms_per_step'])"
