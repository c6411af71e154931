# stage-B shared layouts (MD_PLANE_B_MODE 0 / 1 / 2, unset = the per-launch pick): hashes + c5
# iteration time + the c4 2D class
for i in 1 2; do for m in 0 1 auto; do
  echo "== MODE=$m"
  if [ $m = auto ]; then E=""; else E="MD_PLANE_B_MODE=$m"; fi
  env $E timeout 300 python scripts/plane_adj_probe.py 2>&1 | cut -c1-45 | tail -13
  env $E timeout 300 python scripts/c4_2d_probe.py 1024 2>&1 | tail -1
done; done
