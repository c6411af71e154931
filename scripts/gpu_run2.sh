set -x
timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_f32.log 2>&1; echo "bench32 rc=$?"
tail -1 gpurun_out/bench_f32.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --dtype float64 > gpurun_out/bench_f64.log 2>&1; echo "bench64 rc=$?"
tail -1 gpurun_out/bench_f64.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --batch 512 --e2e-batch 16"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_iter_lines_fast -s 3 -c 1 -o gpurun_out/prof_iterfast_f32 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
