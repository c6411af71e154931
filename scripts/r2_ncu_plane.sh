# ncu --set full of one c5 iteration's plane stage kernels (k_plane_a_fast / k_plane_b_fast)
T=${1:-r2pl}
O=gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_plane" -c 2 -o $O/${T}_prof python scripts/c5_probe.py 16384 > $O/${T}_ncu.log 2>&1; echo "ncu rc=$?"
