# GPU test pass: the whole -m gpu suite + smoke(); run via gpurun.
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -20
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
