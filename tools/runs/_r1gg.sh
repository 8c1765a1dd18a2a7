#!/bin/bash
# small D = 2, 3 transforms (warp-block, batch adjoints, cell-mode interp); compute-sanitizer is closed on the pool (exit 86)
out=gpurun_out/r01gg; mkdir -p $out
timeout 300 python tools/sanitize_small.py > $out/plain.log 2>&1; echo "exit $?" >> $out/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize_small.py > $out/$tool.log 2>&1
  echo "exit $?" >> $out/$tool.log
done
