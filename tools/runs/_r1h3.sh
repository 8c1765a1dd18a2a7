#!/bin/bash
# ncu --set full of the D >= 2 resampling kernels at HEAD (3D, 2D, radial sigma = 2)
out=gpurun_out/r01h3; mkdir -p $out
timeout 300 python tools/prof_stage.py adj_spread,fwd_interp cfg4_3d_64:4 cfg3_2d_512:4 cfg5_radial_s2:4 > $out/plain.log 2>&1; rc=$?
echo "plain exit $rc" >> $out/plain.log
if [ $rc -eq 0 ]; then
  PROF_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread_wb|spread_rowbatch|interp_cell|permute_f|transpose_bm" -c 12 \
     -o $out/full python tools/prof_stage.py adj_spread,fwd_interp cfg4_3d_64:4 cfg3_2d_512:4 cfg5_radial_s2:4 > $out/ncu.log 2>&1
  ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
  ncu -i $out/full.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
fi
rm -f $out/full.ncu-rep
ls -la $out
