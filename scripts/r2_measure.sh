# Full measurement pass: bench lines for every workload + the reference arms (round 2)
# usage: bash scripts/r2_measure.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-r2m}
O=gpurun_out
python bench.py > $O/${T}_bench_c1.json 2> $O/${T}_bench_c1.err; echo "c1 f64 rc=$?"
python bench.py --config c4 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "c4 f64 rc=$?"
python bench.py --config c5 --steps 5 --warmup 3 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err; echo "c5 rc=$?"
python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err; echo "ref rc=$?"
python bench.py --impl reference --config c4 > $O/${T}_bench_ref_c4.json 2> $O/${T}_bench_ref_c4.err; echo "ref c4 rc=$?"
python scripts/c4_breakdown.py float64 > $O/${T}_c4_breakdown_f64.txt 2>&1; echo "c4 breakdown rc=$?"
