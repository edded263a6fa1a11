#!/bin/bash
# Build bisection variants of the FC kernel (skinny_cluster) as separate libs
# under build/ (development aid; wrong results by design): build/lib_fcN.so
set -e
P=paper_2405_05118_b200
make -s -C $P
OBJS=$(ls $P/build/*.o $P/build/kernels/*.o | grep -v kernels/contraction)
for v in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -DMDHB_FC_BISECT=$v -x cu -c $P/csrc/kernels/contraction.cu -o build/contraction_fc$v.o &
done
wait
for v in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/lib_fc$v.so $OBJS build/contraction_fc$v.o -ldl -lpthread
done
