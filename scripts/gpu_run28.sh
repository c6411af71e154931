timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_gpu.log
timeout 300 python scripts/class_probe.py 2>&1 | tail -2
timeout 300 python scripts/c5_probe.py 2>&1 | tail -3
