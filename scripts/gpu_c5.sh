timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "two_level or c3 or c2" > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_c5.log
timeout 300 python scripts/c5_probe.py 16384 2>&1 | tail -1
