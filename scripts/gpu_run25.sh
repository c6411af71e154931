timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_p.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms_per_step'])"
