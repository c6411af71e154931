# c1 float64 throughput per forced cluster size (MD_F64_CLUSTER), two runs each
for cl in 0 8 9 10 ${CLS}; do
  for i in 1 2; do
    MD_F64_CLUSTER=$cl timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-extras --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cl=$cl', round(d['value']), d['stage_ms_per_step'], d['roofline'].get('launch_geometry'))"
  done
done
