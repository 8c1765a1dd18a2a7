mkdir -p gpurun_out/r01s
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01s/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cl_|1c_kernel" -s 12 -c 6 \
    -o gpurun_out/r01s/full python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01s/ncu.log 2>&1
ncu -i gpurun_out/r01s/full.ncu-rep --page details > gpurun_out/r01s/details.txt 2>/dev/null
ncu -i gpurun_out/r01s/full.ncu-rep --page raw --csv > gpurun_out/r01s/raw.csv 2>/dev/null
for k in cl_count cl_scan cl_place cl_fix interp1c spread1c; do
ncu -i gpurun_out/r01s/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01s/src_$k.csv 2>/dev/null
done
