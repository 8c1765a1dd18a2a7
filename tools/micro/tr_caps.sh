mkdir -p gpurun_out/trc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -o /tmp/trace1d tools/micro/trace1d.cu
for c in 2 3 4 7; do echo "cap $c" >> gpurun_out/trc/tr.txt; S1CAP=$c /tmp/trace1d 4 flushed | head -2 | cut -c 1-400 >> gpurun_out/trc/tr.txt; done
tools/quick_bench.sh gpurun_out/trc cfg2_1d_2e18 > gpurun_out/trc/summary.txt 2>&1
