FP_FRAMES=256 timeout 120 python scripts/fp_probe.py > gpurun_out/fp_plain.log 2>&1 && \
FP_FRAMES=256 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fft2" -c 3 -o gpurun_out/prof_fft2_c4 python scripts/fp_probe.py > gpurun_out/ncu_fft2.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_fft2.log
