timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python scripts/c5_probe.py 16384 2>&1 | grep "{"
timeout 300 python scripts/c3_probe.py 2>&1 | tail -1
FP_FRAMES=1024 timeout 120 python scripts/fp_probe.py
timeout 300 python scripts/class_probe.py 2>&1 | grep "c4\[16\]\|c4\[17\]"
