python scripts/c3_probe.py > gpurun_out/c3_plain.log 2>&1 && \
C3_FRAMES=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fft2" -s 20 -c 4 -o gpurun_out/prof_c3 python scripts/c3_probe.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/c3_plain.log
