#!/bin/bash
# Microbenchmarks on the GPU box (built in /tmp, not shipped): FMA peaks and
# the legacy cuFFT callback probe. Usage: tools/gpu_micro.sh <outdir>
out=${1:-gpurun_out/micro}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1; nproc >> $out/lscpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fma_peak tools/micro/fma_peak.cu > $out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=true -o /tmp/cufft_legacy_cb tools/micro/cufft_legacy_cb.cu \
   -L/usr/local/cuda/lib64 -lcufft_static -lculibos >> $out/build.log 2>&1
# clocks sampled while the FMA kernels run
(for i in $(seq 1 40); do nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active --format=csv,noheader; sleep 0.05; done) > $out/fma_clocks.txt 2>&1 &
for r in 1 2 3; do timeout 60 /tmp/fma_peak; done > $out/fma_peak.jsonl 2>&1
wait
timeout 300 /tmp/cufft_legacy_cb > $out/cufft_legacy_cb.jsonl 2>&1; echo "rc $?" >> $out/cufft_legacy_cb.jsonl
