python scripts/c5_probe.py 4096 > gpurun_out/c5p_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_plane" -s 4 -c 2 -o gpurun_out/prof_plane64 python scripts/c5_probe.py 4096 > gpurun_out/ncu_plane.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/c5p_plain.log
