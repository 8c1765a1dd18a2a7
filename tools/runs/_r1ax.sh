mkdir -p gpurun_out/r01ax
python tools/stage_bench.py cfg5_radial_s2 4 auto > gpurun_out/r01ax/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread_rowbatch|interp_cell" -s 1 -c 2 \
    -o gpurun_out/r01ax/full python tools/stage_bench.py cfg5_radial_s2 4 auto > gpurun_out/r01ax/ncu.log 2>&1
ncu -i gpurun_out/r01ax/full.ncu-rep --page details > gpurun_out/r01ax/details.txt 2>/dev/null
for k in spread_rowbatch interp_cell; do
ncu -i gpurun_out/r01ax/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01ax/src_$k.csv 2>/dev/null
done
