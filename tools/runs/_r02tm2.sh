set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_size_invariance" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
for w in resnet50 sweep:1e6:50; do
  echo "== ab $w"; timeout 600 python tools/ab_time.py liblars_b200_head.so liblars_b200_notmem.so liblars_b200.so --workload $w --reps 2 2>&1 | tail -3
done
