set -u
for cb in 8 4 2 1; do
  echo "== chunk $cb"
  LARS_CHUNK_BATCHES=$cb timeout 600 python tools/shard_time.py --workloads resnet50,alexnet_bn,sweep:1e6:50 --worlds 1,4,8 --reps 20 2>&1 | grep -v summary | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['workload'], 'P', d['P'], 't_max', d['t_max_us'], 'E_k', d.get('E_k'))"
done
for g in 148 222; do
  echo "== grid $g"
  timeout 600 python tools/shard_time.py --workloads resnet50,sweep:1e6:50 --worlds 1,8 --reps 20 --grid $g 2>&1 | grep -v summary | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['workload'], 'P', d['P'], 't_max', d['t_max_us'], 'E_k', d.get('E_k'))"
done
