python scripts/c5_probe.py 16384 > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_subfft|k_big_wiener|k_plane" -c 6 -o gpurun_out/prof_c5 python scripts/c5_probe.py 16384 > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_c5.log
