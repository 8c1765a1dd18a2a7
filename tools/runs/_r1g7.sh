#!/bin/bash
# spread_wb warps per CTA sweep (NFFTB_WB_WARPS = 1, 2, 4, 8), 2D and 3D; parity subset
out=gpurun_out/r01g7; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -x -q -k "warp_block or full_size" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for w in 1 2 4 8; do
  for cfg in cfg3_2d_512 cfg4_3d_64; do
    echo "warps $w" >> $out/stages.log
    NFFTB_WB_WARPS=$w STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
  done
done
