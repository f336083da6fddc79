# A/B of several library builds: ab_multi.sh ROUNDS TAG...
rounds=$1; shift
for round in $(seq $rounds); do
for v in "$@"; do
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 2 65536 4
  python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$v.so 4 16384 4
done; done
