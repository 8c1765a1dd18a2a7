#!/bin/bash
# quick per-config bench lines (diagnostic): tools/quick_bench.sh <out> cfg...
out=$1; shift; mkdir -p $out
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps ${QSTEPS:-30} --warmup 5 --no-configs --no-sweep --no-cpu --no-e2e --no-strategies > $out/b_$c.log 2>&1
  python tools/bench_summary.py $out/b_$c.log 2>&1 | head -3 | sed "s/^/$c: /"
done
