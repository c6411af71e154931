timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_f32.log 2>&1; echo "bench32 rc=$?"
tail -1 gpurun_out/bench_f32.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --dtype float64 > gpurun_out/bench_f64.log 2>&1; echo "bench64 rc=$?"
tail -1 gpurun_out/bench_f64.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "benchref rc=$?"
tail -1 gpurun_out/bench_ref.log
lscpu | grep -E "Model name|^CPU\(s\)"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --batch 1024 --e2e-batch 64"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
