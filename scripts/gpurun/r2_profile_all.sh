#!/bin/bash
# ncu --set full of every library kernel on a BASELINE-shaped workload (one launch each; the plain run
# first, ncu only after it exited 0).  Usage: r2_profile_all.sh [WORKLOAD...]
mkdir -p gpurun_out/prof
declare -A K=([cfg0]=locus_warp_kernel [cfg1]=locus_kernel [cfg2]=locus_warp_kernel [bench2]=locus_warp_kernel [cfg3]=locus_warp_kernel
              [cfg4]=locus_warp_kernel [cfg4f32]=locus_warp_kernel [warm2]=locus_warp_kernel
              [brute1]=brute_thread_kernel [brute0]=brute_chunk_kernel [lp2]=lp_simplex_kernel
              [cert2]=axiswise_minimum_kernel [gen4]=gen_kernel [genspec]=genspec_kernel)
works=${@:-cfg0 cfg1 cfg2 bench2 cfg3 cfg4 cfg4f32 warm2 brute1 brute0 lp2 cert2 gen4 genspec}
for w in $works; do
  if timeout 600 python scripts/prof_kernels.py $w --units gpurun_out/prof/units_$w.json > gpurun_out/prof/plain_$w.log 2>&1; then
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:${K[$w]} -s 1 -c 1 \
      -f -o gpurun_out/prof/prof_$w python scripts/prof_kernels.py $w > gpurun_out/prof/ncu_$w.log 2>&1
    echo "$w ncu rc=$?"
  else
    echo "$w plain run failed"; tail -3 gpurun_out/prof/plain_$w.log
  fi
done
