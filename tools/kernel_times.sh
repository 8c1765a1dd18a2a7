#!/bin/bash
# usage: tools/kernel_times.sh <config> <m> <method> <out.csv> [kernel-regex]  (run on the GPU box)
python tools/stage_bench.py $1 $2 $3 > gpurun_out/plain_kt.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,smsp__inst_executed.sum \
    --clock-control none --cache-control none -k regex:"${5:-.}" -s 60 -c 24 --csv --log-file $4 python tools/stage_bench.py $1 $2 $3 > /dev/null 2>&1
