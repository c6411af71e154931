./scripts/probes/cluster_geom > gpurun_out/r2e_geom.txt 2>&1; echo "geom rc=$?"
bash scripts/gpu_variants.sh base nw16 > gpurun_out/r2e_variants.txt 2>&1; echo "variants rc=$?"
