# interleaved A/B of plane-kernel variants: base, TAG, base, TAG (c5 bench + c4 2D class)
for t in base "$1" base "$1"; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  c5=$(MD_LIB=$L timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), d['clocks']['sm_mhz'])")
  c4=$(MD_LIB=$L timeout 600 python scripts/c4_breakdown.py float64 2>&1 | grep "fourier2d per-it" | awk "{print \$5}")
  echo "$t c5 $c5 c4-2D $c4"
done
