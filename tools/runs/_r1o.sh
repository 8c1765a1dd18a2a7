mkdir -p gpurun_out/r01o
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01o/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01o/pytest_gpu.log
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01o/stage_q.log 2>&1
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01o/stage_q.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-sweep > gpurun_out/r01o/bench.log 2>&1
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01o/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"cb_|1c_kernel" -s 8 -c 16 --csv --log-file gpurun_out/r01o/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto > /dev/null 2>&1
