timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
timeout 300 python scripts/class_probe.py 2>&1 | tail -10
