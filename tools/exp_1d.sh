#!/bin/bash
# 1D step experiments (diagnostic): grid caps / priorities -> one bench line each
out=${1:-gpurun_out/exp}; mkdir -p $out
for s1 in ${S1LIST:-4 5 6}; do for i1 in ${I1LIST:-0}; do for pr in ${PRLIST:-1}; do
  NFFTB_X_S1CAP=$s1 NFFTB_X_I1CAP=$i1 NFFTB_ADJ_PRIORITY=$pr timeout 300 python bench.py --steps 100 --warmup 5 --no-configs --no-sweep --no-cpu --no-e2e > $out/b_${s1}_${i1}_${pr}.log 2>&1
  python - $out/b_${s1}_${i1}_${pr}.log $s1 $i1 $pr <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2:], 'FAILED'); sys.exit()
d=json.loads(l[0])
print('s1cap',sys.argv[2],'i1cap',sys.argv[3],'prio',sys.argv[4],'step_us %.1f'%(d['ms_per_step']*1e3), 'seq %.1f'%(d['ms_per_step_sequential_no_events']*1e3), {k:round(v*1e3,1) for k,v in d['stages_ms_marginal'].items()})
PY
done; done; done
