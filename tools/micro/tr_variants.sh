#!/bin/bash
# Timeline variants of the D = 1 kernels (diagnostic): tools/micro/tr_variants.sh <out> "<flags1>" "<flags2>" ...
out=$1; shift
mkdir -p $out
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include $v -o /tmp/trace1d tools/micro/trace1d.cu || continue
  for mode in flushed warm; do echo "== $v $mode S1CAP=$S1CAP" >> $out/tr.json; /tmp/trace1d 4 $mode | head -3 >> $out/tr.json; done
done
