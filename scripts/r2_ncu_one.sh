# one ncu --set full capture of the c1 iteration kernel (after a plain run exits 0)
T=${1:-r2}
O=gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-extras --batch 1024 --e2e-batch 64"
$CMD > $O/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines64" -s 1 -c 1 -o $O/${T}_prof $CMD > $O/${T}_ncu.log 2>&1; echo "ncu rc=$?"
