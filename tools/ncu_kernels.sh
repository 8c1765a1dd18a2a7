#!/bin/bash
# ncu --set full of selected kernels (GPU box): tools/ncu_kernels.sh <outdir> <kernel-regex> <count> <cmd...>
out=$1; rx=$2; cnt=$3; shift 3
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt -o /tmp/ncu_full_$$ "$@" > $out/ncu.log 2>&1
ncu -i /tmp/ncu_full_$$.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
ncu -i /tmp/ncu_full_$$.ncu-rep --page details --csv > $out/full_details.csv 2>/dev/null
ncu -i /tmp/ncu_full_$$.ncu-rep --page source --csv --print-source sass > $out/full_source.csv 2>/dev/null
ls -la $out
