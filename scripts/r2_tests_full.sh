# the whole GPU suite (+ durations), then smoke
O=gpurun_out
T=${1:-r2t}
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > $O/${T}_pytest_all.log 2>&1; echo "pytest all rc=$?"; tail -3 $O/${T}_pytest_all.log
