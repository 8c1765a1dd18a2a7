mkdir -p gpurun_out/r01ak
for i in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01ak/bench_fused$i.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e --no-fused > gpurun_out/r01ak/bench_plain$i.log 2>&1
done
timeout 600 python bench.py --config cfg3_2d_512 --steps 50 --warmup 5 --no-cpu --no-sweep --no-e2e > gpurun_out/r01ak/bench2d_fused.log 2>&1
timeout 600 python bench.py --config cfg3_2d_512 --steps 50 --warmup 5 --no-cpu --no-sweep --no-e2e --no-fused > gpurun_out/r01ak/bench2d_plain.log 2>&1
