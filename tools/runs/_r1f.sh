mkdir -p gpurun_out/r01f
python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01f/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"interp1d|spread1d|binsort" -s 3 -c 3 \
    -o gpurun_out/r01f/full python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01f/ncu.log 2>&1
for k in interp1d spread1d binsort; do
ncu -i gpurun_out/r01f/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01f/src_$k.csv 2>/dev/null
done
ncu -i gpurun_out/r01f/full.ncu-rep --page raw --csv > gpurun_out/r01f/full_raw.csv 2>/dev/null
