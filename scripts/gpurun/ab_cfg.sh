#!/bin/bash
# same-box A/B of library builds: ab_cfg.sh CONFIG B ROUNDS TAG... (libladlasso_b200_TAG.so)
cfg=$1; B=$2; rounds=$3; shift 3
for r in $(seq $rounds); do
  for t in "$@"; do timeout 600 python scripts/ab_timing.py paper_2510_15649_b200/libladlasso_b200_$t.so $cfg $B 3; done
done
