for g in 296 222 148 74; do
  echo "== grid $g"
  timeout 600 python tools/shard_time.py --workloads sweep:1e6:50,resnet50 --worlds 1,8 --grid $g --reps 20 2>&1 | grep '"P"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['workload'], 'P', d['P'], 'grid', d['grid'], 't_max_us', d['t_max_us'], 'frac', d['frac_hbm_max'])"
done
