# Full measurement pass: bench lines for every workload + ncu launch list + full captures.
# usage: bash scripts/gpu_measure.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-r1}
O=gpurun_out
python bench.py > $O/${T}_bench_c1.json 2> $O/${T}_bench_c1.err; echo "c1 rc=$?"
python bench.py --dtype float64 --no-cpu > $O/${T}_bench_f64.json 2> $O/${T}_bench_f64.err; echo "f64 rc=$?"
python bench.py --config c4 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "c4 rc=$?"
python bench.py --config c5 --steps 5 --warmup 3 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err; echo "c5 rc=$?"
python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err; echo "ref rc=$?"
python bench.py --impl reference --config c4 > $O/${T}_bench_ref_c4.json 2> $O/${T}_bench_ref_c4.err; echo "ref c4 rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --batch 1024 --e2e-batch 64"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches_c1.csv $CMD > $O/ncu_l.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_fused_lines|k_wiener_lines" -s 2 -c 2 -o $O/${T}_prof_c1 $CMD > $O/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
FP_FRAMES=256 python scripts/fp_probe.py > $O/plain2.log 2>&1 && \
FP_FRAMES=256 ncu --set full --clock-control none --import-source on -k regex:"k_fused_plane|k_fft2" -s 2 -c 4 -o $O/${T}_prof_c4_2d python scripts/fp_probe.py > $O/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
