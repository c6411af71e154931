# stage A/B plane kernels: in-tree vs a variant library (arg: TAG of variants/libmdcuda_TAG.so)
for L in "" variants/libmdcuda_$1.so; do
  echo "== lib ${L:-in-tree}"
  MD_LIB=$L timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d.get('stage_ms_per_step'))"
  MD_LIB=$L timeout 600 python scripts/c4_breakdown.py float64 2>&1 | tail -4
done
