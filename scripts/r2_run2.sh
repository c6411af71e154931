O=gpurun_out
bash scripts/r2_check.sh r2c
timeout 600 python -m pytest tests/test_gpu_fused64.py -q -m gpu > $O/r2c_fused64.log 2>&1; echo "fused64 tests rc=$?"
