timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "bench c1 rc=$?"
tail -1 gpurun_out/bench_c1.log
timeout 600 python bench.py --config c4 --steps 10 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -3 gpurun_out/bench_c4.log
timeout 400 python bench.py --impl reference --config c4 --steps 3 --warmup 1 > gpurun_out/bench_ref_c4.log 2>&1; echo "ref c4 rc=$?"
tail -1 gpurun_out/bench_ref_c4.log
