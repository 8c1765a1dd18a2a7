mkdir -p gpurun_out/r01j
python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01j/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread1d|binsort|interp1d" -s 3 -c 3 \
    -o gpurun_out/r01j/full python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01j/ncu.log 2>&1
for k in interp1d spread1d binsort; do
ncu -i gpurun_out/r01j/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01j/src_$k.csv 2>/dev/null
done
ncu -i gpurun_out/r01j/full.ncu-rep --page details > gpurun_out/r01j/details.txt 2>/dev/null
