O=gpurun_out
for cfg in "4096 8 1" "8192 8 1" "16384 2 1 slabs" "16384 8 1 single" "16384 8 0 slabs" "16384 8 1 slabs"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/slab_probe.py $cfg > $O/r2u_slab_$(echo $cfg | tr ' ' _).log 2>&1; echo "$cfg rc=$?"; tail -2 $O/r2u_slab_$(echo $cfg | tr ' ' _).log
done
