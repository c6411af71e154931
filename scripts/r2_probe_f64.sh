# f64 c1 baseline lines (per-iteration and the existing cluster kernel) + ncu capture of both
O=gpurun_out
python bench.py --dtype float64 --steps 10 --warmup 3 --no-cpu > $O/r2a_f64.json 2> $O/r2a_f64.err; echo "f64 rc=$?"
python bench.py --dtype float64 --fused on --steps 10 --warmup 3 --no-cpu > $O/r2a_f64_fused.json 2> $O/r2a_f64_fused.err; echo "f64 fused rc=$?"
CMD="python bench.py --dtype float64 --steps 1 --warmup 1 --no-cpu --batch 512 --e2e-batch 16"
ncu --set full --clock-control none --import-source on -k regex:"k_iter_lines_fast" -s 1 -c 1 -o $O/r2a_prof_f64 $CMD > $O/r2a_ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines" -s 1 -c 1 -o $O/r2a_prof_f64_fused $CMD --fused on > $O/r2a_ncu2.log 2>&1; echo "ncu2 rc=$?"
