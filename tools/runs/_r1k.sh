#!/bin/bash
# end-of-session evidence at HEAD: gpu tests, smoke, bench + ncu (tools/gpu_round.sh), per-config bench lines
bash tools/gpu_round.sh r01k
bash tools/config_sweep.sh gpurun_out/r01k/sweep
ls -la gpurun_out/r01k/sweep
