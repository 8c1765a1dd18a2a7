#!/bin/bash
# ncu --set full of the batch adjoint (radial)
out=gpurun_out/r01g2; mkdir -p $out
timeout 300 python tools/prof_stage.py adj_spread cfg5_radial_s2:4 > $out/plain.log 2>&1; rc=$?
echo "plain exit $rc" >> $out/plain.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread_rowbatch|transpose_bm" -c 3 \
     -o $out/full python tools/prof_stage.py adj_spread cfg5_radial_s2:4 > $out/ncu.log 2>&1
  ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
  ncu -i $out/full.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
fi
rm -f $out/full.ncu-rep
ls -la $out
