# stage B adjacent-column variants (MD_PLANE_ADJ 0 / 1 / 2 / 3): hashes + c5 time + c4 2D class
for i in 1 2; do for m in 0 1 2 3; do
  echo "== ADJ=$m"
  MD_PLANE_ADJ=$m timeout 300 python scripts/plane_adj_probe.py 2>&1 | cut -c1-45 | tail -13
  MD_PLANE_ADJ=$m timeout 300 python scripts/c4_2d_probe.py 1024 2>&1 | tail -1
done; done
