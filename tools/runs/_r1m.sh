mkdir -p gpurun_out/r01m
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01m/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"interp1c|spread1c|cellsort|binsort" -s 4 -c 4 \
    -o gpurun_out/r01m/full python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01m/ncu.log 2>&1
for k in interp1c spread1c cellsort binsort; do
ncu -i gpurun_out/r01m/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01m/src_$k.csv 2>/dev/null
done
ncu -i gpurun_out/r01m/full.ncu-rep --page raw --csv > gpurun_out/r01m/full_raw.csv 2>/dev/null
ncu -i gpurun_out/r01m/full.ncu-rep --page details > gpurun_out/r01m/details.txt 2>/dev/null
