# stage A/B plane kernels: in-tree vs variant libraries (args: TAGs of variants/libmdcuda_TAG.so)
for t in base "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  echo "== $t"
  MD_LIB=$L timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'])"
  MD_LIB=$L timeout 600 python scripts/c4_breakdown.py float64 2>&1 | tail -2
done
