# launch list (durations) of one 16384^2 Wiener (scripts/fft_ab_probe.py FFT_AB_PROFILE=1)
FFT_AB_PROFILE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_wiener_launches.csv python scripts/fft_ab_probe.py > gpurun_out/r2_wiener_launches.log 2>&1
echo rc=$?
