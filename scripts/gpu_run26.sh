timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
FP_FRAMES=1024 timeout 120 python scripts/fp_probe.py
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-200
