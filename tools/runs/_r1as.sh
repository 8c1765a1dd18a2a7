mkdir -p gpurun_out/r01as
timeout 900 python -m pytest tests -m gpu -x -q -k "1d or config1 or cfg2 or batch_and" > gpurun_out/r01as/pytest.log 2>&1; echo exit $? >> gpurun_out/r01as/pytest.log
for s1 in 0 296 444 592 888; do for i1 in 0 592; do
echo "s1=$s1 i1=$i1" >> gpurun_out/r01as/chain.log
NFFTB_S1_CTAS=$s1 NFFTB_I1_CTAS=$i1 python tools/chain_times.py >> gpurun_out/r01as/chain.log 2>&1
done; done
