#!/bin/bash
# Round evidence on one GPU box: tests, smoke, the default bench line, the ncu
# launch list of the bench command and ncu --set full of the dominant kernels of
# every config. Usage: tools/gpu_evidence.sh <outdir>
out=${1:-gpurun_out/evidence}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 1200 python bench.py > $out/bench.log 2>&1; rc=$?; echo "bench exit $rc" >> $out/bench.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu --no-configs --no-strategies > $out/ncu_launches.log 2>&1
  for cfg in cfg2_1d_2e18 cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2 cfg5_radial_s125; do
    tools/ncu_kernels.sh $out/full_$cfg "interp|spread|transpose|permute|correct" 6 python tools/stage_bench.py $cfg 4 > /dev/null 2>&1
    rm -f $out/full_$cfg/full_source.csv
  done
fi
ls -la $out
