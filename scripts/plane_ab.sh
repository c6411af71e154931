# plane stage kernels per library variant: hashes + c5 iteration time (plane_adj_probe.py) and the
# c4 2D class (c4_2d_probe.py):  bash scripts/plane_ab.sh "base TAG ..."
for i in 1 2; do for t in $1; do
  if [ "$t" = base ]; then L=""; else L="variants/libmdcuda_$t.so"; fi
  echo "== $t"; MD_LIB=$L timeout 300 python scripts/plane_adj_probe.py 2>&1 | cut -c1-45 | tail -13
  MD_LIB=$L timeout 300 python scripts/c4_2d_probe.py 1024 2>&1 | tail -1
done; done
