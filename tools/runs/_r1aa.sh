mkdir -p gpurun_out/r01aa
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r01aa/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01aa/ref.log 2>&1
