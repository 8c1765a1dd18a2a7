#!/bin/bash
out=gpurun_out/r01gb; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -x -q -k "warp_block" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
