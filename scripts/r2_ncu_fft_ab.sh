# ncu --set full of the 16384^2 Wiener's two-level passes, per library variant (args: TAG=LIB ...)
for tl in "$@"; do
  t=${tl%%=*}; L=${tl#*=}
  MD_LIB=$L FFT_AB_PROFILE=1 timeout 600 ncu --set full --clock-control none -k regex:k_subfft -c 6 \
    -o gpurun_out/r2fft_$t -f python scripts/fft_ab_probe.py > gpurun_out/r2fft_$t.log 2>&1
  echo "$t rc=$?"
done
