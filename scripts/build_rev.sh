#!/bin/bash
# Build the C-ABI library of git revision $1 into paper_2510_15649_b200/libladlasso_b200_$2.so (A/B timing).
set -e
rev=$1; tag=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/include" "$tmp/a/b/csrc"
git -C "$root" show "$rev:include/ladlasso_b200.h" > "$tmp/include/ladlasso_b200.h"
for f in $(git -C "$root" ls-tree --name-only "$rev" paper_2510_15649_b200/csrc/); do
  git -C "$root" show "$rev:$f" > "$tmp/a/b/csrc/$(basename "$f")"
done
sed -i 's#../../include#../../../include#' "$tmp/a/b/csrc/ladlasso_b200.cu"
flags=$(cd "$root" && python -c "import sys; sys.path.insert(0,'.'); from paper_2510_15649_b200 import _build; print(' '.join(_build.NVCC_FLAGS))")
(cd "$tmp/a/b/csrc" && nvcc $flags -o "$root/paper_2510_15649_b200/libladlasso_b200_$tag.so" ladlasso_b200.cu)
rm -rf "$tmp"
echo "built paper_2510_15649_b200/libladlasso_b200_$tag.so from $rev"
