# c1 (float64) launch list + ncu --set full of the Wiener and fused iteration kernels
# usage: bash scripts/r2_ncu_c1.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-r2}
O=gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-extras --batch 1024 --e2e-batch 64"
$CMD > $O/${T}_plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c1.csv $CMD > $O/${T}_ncu_l.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines64|k_wiener_lines" -s 2 -c 2 -o $O/${T}_prof_c1 $CMD > $O/${T}_ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
