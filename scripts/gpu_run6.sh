timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c4 --steps 10 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -1 gpurun_out/bench_c4.log
