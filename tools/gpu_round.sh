#!/bin/bash
# One GPU-box pass (run via gpurun from the repo root):
#   gpu tests, smoke, bench (plain), ncu launch list of the bench command,
#   one `ncu --set full` capture of the dominant resampling kernels.
# Usage: tools/gpu_round.sh <tag> [bench args...]
tag=${1:-r01}; shift
mkdir -p gpurun_out
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py "$@" > $out/bench.log 2>&1; rc=$?; echo "bench exit $rc" >> $out/bench.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu "$@" > $out/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"interp|spread" -s 4 -c 4 \
      -o $out/full python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu "$@" > $out/ncu_full.log 2>&1
  ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
fi
ls -la $out
