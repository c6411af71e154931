# float64 A/B: c1 per-iteration and fused, c5 probe, per library variant ("base" = in-tree)
for t in "$@"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  for fu in auto on; do MD_LIB=$L timeout 300 python bench.py --dtype float64 --fused $fu --steps 10 --warmup 3 --no-cpu --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t f64 fused=$fu', round(d['value']), d['stage_ms_per_step'])"; done
  MD_LIB=$L timeout 300 python scripts/c5_probe.py 16384 2>&1 | tail -1 | sed "s/^/$t c5 /"
done
