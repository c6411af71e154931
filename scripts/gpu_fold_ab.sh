# A/B of the folded-1/wi box update against the committed library (variants/libmdcuda_head.so)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for r in 1 2; do for t in head base; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  MD_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $t', round(d['value']), d['stage_ms_per_step'])"
  MD_LIB=$L timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $t', round(d['value']))"
done; done
