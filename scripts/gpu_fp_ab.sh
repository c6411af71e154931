# 2D-PSF frames (c4's 2D class, scripts/fp_probe.py) per library variant ("base" = in-tree)
for t in "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  MD_LIB=$L FP_FRAMES=1024 timeout 300 python scripts/fp_probe.py 2>&1 | sed "s/^/$t /"
done
