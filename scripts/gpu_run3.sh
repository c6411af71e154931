set -x
timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_f32.log 2>&1; echo "bench32 rc=$?"
tail -1 gpurun_out/bench_f32.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --dtype float64 > gpurun_out/bench_f64.log 2>&1; echo "bench64 rc=$?"
tail -1 gpurun_out/bench_f64.log
