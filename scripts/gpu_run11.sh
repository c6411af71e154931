CMD="python bench.py --steps 3 --warmup 1 --no-cpu --batch 1024 --e2e-batch 64"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines|k_wiener_lines_reg" -s 2 -c 2 -o gpurun_out/prof_r1_c1b $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -1 gpurun_out/plain.log
