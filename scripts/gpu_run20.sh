timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "fused_plane" -x > gpurun_out/pytest_fp.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_fp.log
timeout 300 python scripts/class_probe.py 2>&1 | tail -12
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -2 | cut -c1-600
