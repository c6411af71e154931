timeout 500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "two_level or f2d" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/c5_probe.py; echo "c5 rc=$?"
