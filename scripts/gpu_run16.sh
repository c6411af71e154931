python scripts/plane_probe.py c4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_plane_|k_fft2" -s 4 -c 4 -o gpurun_out/prof_plane_c4 python scripts/plane_probe.py c4 > gpurun_out/ncu1.log 2>&1; echo "ncu c4 rc=$?"
python scripts/plane_probe.py c2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_plane_" -s 2 -c 2 -o gpurun_out/prof_plane_c2 python scripts/plane_probe.py c2 > gpurun_out/ncu2.log 2>&1; echo "ncu c2 rc=$?"
