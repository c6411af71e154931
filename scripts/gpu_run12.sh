timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
tail -1 gpurun_out/bench_c1.log
timeout 300 python bench.py --no-cpu --dtype float64 --fused on > gpurun_out/bench_c1_f64.log 2>&1; echo "c1 f64 fused rc=$?"
tail -1 gpurun_out/bench_c1_f64.log
