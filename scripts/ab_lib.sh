# A/B of library variants on c1 float64: bash scripts/ab_lib.sh "tagA tagB ..." [bench args]
# tag "base" = the regular in-tree build; others = variants/libmdcuda_TAG.so
TAGS=${1:-base}; shift
for i in 1 2 3; do
  for t in $TAGS; do
    if [ "$t" = base ]; then L=""; else L="variants/libmdcuda_$t.so"; fi
    MD_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-extras --e2e-batch 64 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value']), {k: round(v, 3) for k, v in d['stage_ms_per_step'].items()})"
  done
done
