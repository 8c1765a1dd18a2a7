mkdir -p gpurun_out/r01t
./tools/micro/short_kernels > gpurun_out/r01t/micro.log 2>&1
for s in 1 2 3 4; do NFFTB_DIAG_PRE_STOP=$s timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01t/pre.log 2>&1; done
for s in 1 2 3 4; do NFFTB_DIAG_PRE_STOP=$s timeout 300 python tools/stage_bench.py cfg3_2d_512 4 auto >> gpurun_out/r01t/pre.log 2>&1; done
