# c4 (65536 frames, float64): PSF groups over 2 / 3 / 4 streams (MD_C4_STREAMS)
for i in 1 2; do for cfg in "2 round_robin" "3 round_robin" "4 round_robin"; do set -- $cfg
  MD_C4_STREAMS=$1 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-extras --e2e-batch 64 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['ms_per_step'], 2))"
done; done
