# smoke + fused / parity tests + a short default bench (no extras)
O=gpurun_out
T=${1:-r2q}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_fused64.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q -m gpu > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/${T}_pytest.log
timeout 600 python bench.py --no-cpu --no-extras > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$O/${T}_bench.json').read()); print(round(d['value']), d['stage_ms_per_step'], d['plan'])"
