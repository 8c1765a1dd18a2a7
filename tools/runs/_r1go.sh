#!/bin/bash
# spread_wb launch bounds (128, 5) probe (96 regs, spills: 3D 279 vs 234 us, not kept)
out=gpurun_out/r01go; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "warp_block or full_size or seam" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg4_3d_64; do STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1; done
