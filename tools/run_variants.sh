#!/bin/bash
# Library variants (diagnostic): tools/run_variants.sh <out> <cfg...>; each variants/libnfft_*.so in turn (REPEAT times)
out=$1; shift; mkdir -p $out
cp paper_2208_00049_b200/libnfft_b200.so /tmp/lib_orig.so
for rep in $(seq 1 ${REPEAT:-1}); do
for v in variants/libnfft_*.so; do
  cp $v paper_2208_00049_b200/libnfft_b200.so
  tag=$(basename $v .so)
  tools/quick_bench.sh $out/$tag "$@" | sed "s/^/$tag /" >> $out/summary.txt 2>&1
done
done
cp /tmp/lib_orig.so paper_2208_00049_b200/libnfft_b200.so
