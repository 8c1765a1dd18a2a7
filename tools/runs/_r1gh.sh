#!/bin/bash
# interp1c occupancy probe (launch bounds 256 x 4; interp 8.4 us either way, not kept): 1D stage times and bench line
out=gpurun_out/r01gh; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -x -q -k "1d or config1 or full_size" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto > $out/stages.log 2>&1
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> $out/stages.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-sweep --no-cpu > $out/bench.log 2>&1
