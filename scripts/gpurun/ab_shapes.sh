# A/B of warp-kernel launch shapes (LAD_WARP_WARPS_PER_BLOCK x LAD_WARP_MIN_BLOCKS builds)
python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_w8x4.so 2 4096 1 2>&1 | tail -3
for round in 1 2; do
for v in w7x4 w6x4 w8x3 w7x3; do
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 2 65536 3
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 4 16384 3
done; done
