timeout 600 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_parity.py -q -k "host_paramset or divergence_host or interleaved or reference_style" 2>&1 | tail -2
timeout 600 python tools/host_paramset_time.py --workload resnet50
timeout 600 python tools/host_paramset_time.py --workload alexnet_bn --steps 5
