timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -20
timeout 300 python scripts/class_probe.py 2>&1 | tail -2
timeout 300 python scripts/c5_probe.py 2>&1 | tail -3
