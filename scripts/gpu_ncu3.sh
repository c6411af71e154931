CMD="python bench.py --steps 2 --warmup 1 --no-cpu --batch 1024 --e2e-batch 16"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines|k_wiener_lines" -s 2 -c 2 -o gpurun_out/prof_c1_r1c $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full.log
