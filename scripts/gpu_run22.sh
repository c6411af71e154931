timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "overlapped or fused" > gpurun_out/pytest_ov.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_ov.log
for ov in 0 1; do
  MD_OVERLAP=$ov timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-400
  MD_OVERLAP=$ov timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
done
