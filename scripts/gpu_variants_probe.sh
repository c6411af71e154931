# pipe_probe per library variant: bash scripts/gpu_variants_probe.sh TAG...  ("base" = in-tree)
for t in "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  echo "== $t"; MD_LIB=$L timeout 300 python scripts/pipe_probe.py 2>&1 | tail -6
done
