mkdir -p gpurun_out/r01at
for s1 in 0 888 592; do for rep in 1 2; do
NFFTB_S1_CTAS=$s1 timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01at/b_${s1}_$rep.log 2>&1
done; done
