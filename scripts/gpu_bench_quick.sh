timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for c in c1 c4; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'e2e_f64', round(d['e2e_f64']['value']), 'e2e_u8', round(d['e2e_u8']['value']))"
done
