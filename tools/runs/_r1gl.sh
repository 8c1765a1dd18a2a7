#!/bin/bash
# 1D step vs the spread's resident grid (NFFTB_S1_CTAS) and the interp grid (NFFTB_I1_CTAS)
out=gpurun_out/r01gl; mkdir -p $out
for c in 296 444 592 740 888; do
  echo "S1_CTAS $c" >> $out/bench.log
  NFFTB_S1_CTAS=$c timeout 600 python bench.py --steps 300 --warmup 10 --no-sweep --no-cpu --no-e2e 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step']*1000)" >> $out/bench.log
done
for c in 296 592; do
  echo "I1_CTAS $c" >> $out/bench.log
  NFFTB_I1_CTAS=$c timeout 600 python bench.py --steps 300 --warmup 10 --no-sweep --no-cpu --no-e2e 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step']*1000)" >> $out/bench.log
done
