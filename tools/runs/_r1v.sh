mkdir -p gpurun_out/r01v
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01v/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"1c_kernel|cl_place|cl_scan" -s 8 -c 4 \
    -o gpurun_out/r01v/full python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01v/ncu.log 2>&1
ncu -i gpurun_out/r01v/full.ncu-rep --page details > gpurun_out/r01v/details.txt 2>/dev/null
ncu -i gpurun_out/r01v/full.ncu-rep --page raw --csv > gpurun_out/r01v/raw.csv 2>/dev/null
for k in cl_place cl_scan interp1c spread1c; do
ncu -i gpurun_out/r01v/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01v/src_$k.csv 2>/dev/null
done
