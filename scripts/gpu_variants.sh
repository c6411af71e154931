# c1 iteration time per library variant: bash scripts/gpu_variants.sh TAG...  (MD_LIB=variants/libmdcuda_TAG.so; "base" = in-tree)
for t in "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  for i in 1 2; do MD_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-extras --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value']), d['stage_ms_per_step'])"; done
done
