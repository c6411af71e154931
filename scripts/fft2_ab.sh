# 2D-FFT passes (c4 2D-class Wiener init, c3 convolver) per library variant: bash scripts/fft2_ab.sh "base TAG ..."
for i in 1 2; do for t in $1; do
  if [ "$t" = base ]; then L=""; else L="variants/libmdcuda_$t.so"; fi
  echo "== $t"; MD_LIB=$L timeout 300 python scripts/c4_2d_probe.py 1024 2>&1 | tail -2
  MD_LIB=$L C3_FRAMES=8 timeout 300 python scripts/c3_probe.py 2>&1 | tail -1
done; done
