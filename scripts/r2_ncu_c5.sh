# c5 (16384^2 float64): plain timing, then ncu --set full of the Wiener passes and one iteration's stage kernels
T=${1:-r2c5}
O=gpurun_out
python scripts/c5_probe.py 16384 > $O/${T}_plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/${T}_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_subfft|k_plane" -c 9 -o $O/${T}_prof python scripts/c5_probe.py 16384 > $O/${T}_ncu.log 2>&1; echo "ncu rc=$?"
