timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "fused_plane or golden or fused" > gpurun_out/pytest_fp.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_fp.log
FP_FRAMES=1024 timeout 120 python scripts/fp_probe.py && \
FP_FRAMES=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_plane -c 1 -o gpurun_out/fp_full python scripts/fp_probe.py > gpurun_out/ncu_fp.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_fp.log
