# A/B of the median neighbour walk (LAD_MEDIAN_WALK_HOPS[_WIDE] builds)
for round in 1 2; do
for v in h0_0 h6_0 h8_0 h12_0 h31_0 h31_8 h31_31; do
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 2 65536 4
  [ "$v" = h0_0 -o "$v" = h31_8 -o "$v" = h31_31 ] && python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 4 16384 4
done; done
