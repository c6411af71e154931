timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fused or golden" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
MD_FUSED_LPW=2 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fused or c1" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest lpw2 rc=$?"
tail -2 gpurun_out/pytest_gpu2.log
timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
tail -1 gpurun_out/bench_c1.log | cut -c1-200; grep -o '"stage_ms_per_step[^}]*}' gpurun_out/bench_c1.log
MD_FUSED_LPW=2 timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/bench_c1_lpw2.log 2>&1; echo "c1 lpw2 rc=$?"
tail -1 gpurun_out/bench_c1_lpw2.log | cut -c1-200; grep -o '"stage_ms_per_step[^}]*}' gpurun_out/bench_c1_lpw2.log
