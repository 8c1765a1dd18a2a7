#!/bin/bash
# interp/spread marginal times per tile (diagnostic): tools/tile_sweep.sh <out> <cfg> <tile>...
out=$1; cfg=$2; shift 2; mkdir -p $out
for t in "$@"; do
  timeout 300 python bench.py --config $cfg --tile $t --steps 20 --warmup 3 --no-configs --no-sweep --no-cpu --no-e2e --no-strategies > $out/b_${cfg}_$t.log 2>&1
  python tools/bench_summary.py $out/b_${cfg}_$t.log 2>&1 | sed -n 3p | sed "s/^/$cfg $t /"
done
