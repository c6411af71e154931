# end-to-end (host buffers) A/B of two libraries on one box: bash scripts/gpu_e2e_ab.sh TAG...
for r in 1 2; do for t in "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  MD_LIB=$L timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $t', round(d['value']), round(d['e2e']['value']))"
  MD_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $t', round(d['value']), round(d['e2e']['value']), round(d['e2e_u8']['value']))"
done; done
