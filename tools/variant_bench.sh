#!/bin/bash
# A/B of experiment builds (GPU box): tools/variant_bench.sh <out> "<configs>" <variant.so>...
# Each variant replaces the library for a parity subset + quick bench, then the product library returns.
out=$1; cfgs=$2; shift 2
mkdir -p $out
cp paper_2208_00049_b200/libnfft_b200.so /tmp/product.so
for v in product "$@"; do
  tag=$(basename $v .so)
  [ "$v" != product ] && cp $v paper_2208_00049_b200/libnfft_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${TESTK:-batch_adjoint or radial_batch}" > $out/t_$tag.log 2>&1
  echo "$tag pytest $?" >> $out/summary.txt
  bash tools/quick_bench.sh $out/qb_$tag $cfgs | sed "s/^/$tag /" >> $out/summary.txt
  cp /tmp/product.so paper_2208_00049_b200/libnfft_b200.so
done
