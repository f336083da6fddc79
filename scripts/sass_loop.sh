#!/bin/bash
# Print the SASS of locus_warp_kernel<5,30,double> from the built library (or $1) and count
# the instructions of the coordinate-step loop (from the sparse-bit test to the loop branch).
lib=${1:-paper_2510_15649_b200/libladlasso_b200.so}
cuobjdump -sass -fun '_ZN3lad17locus_warp_kernelILi5ELi30EdEEvNS_9LocusArgsE' "$lib" > /tmp/k530.sass
wc -l < /tmp/k530.sass
