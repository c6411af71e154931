timeout 600 python scripts/class_probe.py 2>&1 | tail -12
