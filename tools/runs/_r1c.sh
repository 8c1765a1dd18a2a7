mkdir -p gpurun_out/r01c
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01c/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01c/pytest_gpu.log
for rr in 1 2 4 8; do NFFTB_BS_RR=$rr timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto 512 | sed "s/^/rr=$rr /" >> gpurun_out/r01c/stage_rr.log 2>&1; done
for rr in 1 2 4 8; do NFFTB_BS_RR=$rr timeout 300 python tools/stage_bench.py cfg3_2d_512 4 auto | sed "s/^/rr=$rr /" >> gpurun_out/r01c/stage_rr.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 tiled_v1 512 | sed "s/^/v1 /" >> gpurun_out/r01c/stage_rr.log 2>&1
for q in 256 512 1024 2048; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01c/stage_q.log 2>&1; done
