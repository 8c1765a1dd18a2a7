mkdir -p gpurun_out/r01d
python tools/stage_bench.py cfg2_1d_2e18 4 auto 512 > gpurun_out/r01d/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"interp1d|spread1d|binsort|interp_tiled|spread_gather" -s 10 -c 8 \
    -o gpurun_out/r01d/full python tools/stage_bench.py cfg2_1d_2e18 4 auto 512 > gpurun_out/r01d/ncu.log 2>&1
ncu -i gpurun_out/r01d/full.ncu-rep --page raw --csv > gpurun_out/r01d/full_raw.csv 2>/dev/null
ncu -i gpurun_out/r01d/full.ncu-rep --page source --csv -k regex:spread1d > gpurun_out/r01d/src_spread1d.csv 2>/dev/null
ncu -i gpurun_out/r01d/full.ncu-rep --page details > gpurun_out/r01d/details.txt 2>/dev/null
