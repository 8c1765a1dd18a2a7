mkdir -p gpurun_out/r01ao
python tools/stage_bench.py cfg4_3d_64 4 auto > gpurun_out/r01ao/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread_cell|interp_cell" -s 2 -c 2 \
    -o gpurun_out/r01ao/full python tools/stage_bench.py cfg4_3d_64 4 auto > gpurun_out/r01ao/ncu.log 2>&1
ncu -i gpurun_out/r01ao/full.ncu-rep --page details > gpurun_out/r01ao/details.txt 2>/dev/null
for k in interp_cell spread_cell; do
ncu -i gpurun_out/r01ao/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01ao/src_$k.csv 2>/dev/null
done
