#!/bin/bash
out=gpurun_out/r01f4; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "warp_block or batch_adjoint or seam or full_size or radial" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
