mkdir -p gpurun_out/r01ay
timeout 900 python -m pytest tests -m gpu -x -q -k "binning or cell or dense or config1 or 1d" > gpurun_out/r01ay/pytest.log 2>&1; echo exit $? >> gpurun_out/r01ay/pytest.log
for c in 0 148 296 592; do echo "pre_ctas=$c" >> gpurun_out/r01ay/chain.log; NFFTB_PRE_CTAS=$c python tools/chain_times.py >> gpurun_out/r01ay/chain.log 2>&1; done
