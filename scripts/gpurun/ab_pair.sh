# A/B of two library builds: ab_pair.sh TAG_A TAG_B [rounds]
for round in $(seq ${3:-2}); do
for v in $1 $2; do
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 2 65536 4
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 4 16384 4
done; done
