# quick GPU check: smoke, parity + fuzz tests, then the default bench line
O=gpurun_out
T=${1:-r2b}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q -m gpu > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
