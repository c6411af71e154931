timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_p.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_p.log | head
timeout 300 python scripts/c5_probe.py 4096 16384 2>&1 | grep "{"
timeout 300 python scripts/class_probe.py 2>&1 | grep c2
