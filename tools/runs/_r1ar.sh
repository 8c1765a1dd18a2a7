mkdir -p gpurun_out/r01ar
for i in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01ar/bench_prio$i.log 2>&1
NFFTB_ADJ_PRIORITY=0 timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01ar/bench_noprio$i.log 2>&1
done
