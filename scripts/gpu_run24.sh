timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-200
FP_FRAMES=1024 timeout 120 python scripts/fp_probe.py
