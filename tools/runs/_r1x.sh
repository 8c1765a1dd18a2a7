mkdir -p gpurun_out/r01x
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01x/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread1c" -s 8 -c 2 \
    -o gpurun_out/r01x/full python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01x/ncu.log 2>&1
ncu -i gpurun_out/r01x/full.ncu-rep --page details > gpurun_out/r01x/details.txt 2>/dev/null
ncu -i gpurun_out/r01x/full.ncu-rep --page raw --csv > gpurun_out/r01x/raw.csv 2>/dev/null
for k in cl_place cl_scan interp1c spread1c; do
ncu -i gpurun_out/r01x/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01x/src_$k.csv 2>/dev/null
done
