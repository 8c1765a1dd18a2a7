#!/bin/bash
# Fast experiment builds for the 1D kernels: only inst_d1.cu and nfft_api.cu see the -D flags, the other
# objects come from the product build (build/obj). Usage: tools/variant_1d.sh <name> -DNFFTB_...=.. ...
name=$1; shift
o=/tmp/var1d_$name; mkdir -p $o variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -I include"
nvcc $F "$@" -c paper_2208_00049_b200/csrc/inst_d1.cu -o $o/inst_d1.o &
nvcc $F "$@" -c paper_2208_00049_b200/csrc/nfft_api.cu -o $o/nfft_api.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $o/inst_d1.o $o/nfft_api.o build/obj/inst_d2.o build/obj/inst_d3.o \
  -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 && echo "built variants/$name.so"
