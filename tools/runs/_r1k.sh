mkdir -p gpurun_out/r01k
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01k/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01k/pytest_gpu.log
for q in 256 512 1024; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01k/stage_q.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01k/stage_q.log 2>&1
for c in cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01k/stage_q.log 2>&1; done
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01k/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r01k/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto > /dev/null 2>&1
