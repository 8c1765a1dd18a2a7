mkdir -p gpurun_out/r01am
python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01am/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"interp_cell|spread_cell" -s 2 -c 2 \
    -o gpurun_out/r01am/full python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01am/ncu.log 2>&1
ncu -i gpurun_out/r01am/full.ncu-rep --page details > gpurun_out/r01am/details.txt 2>/dev/null
for k in interp_cell spread_cell; do
ncu -i gpurun_out/r01am/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01am/src_$k.csv 2>/dev/null
done
