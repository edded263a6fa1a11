#!/bin/bash
# Build scan_tiles tile-shape variants as separate libs build/lib_scan_<tag>.so
# (development aid): tag=ROUNDSxTHREADSxMINB
set -e
P=paper_2405_05118_b200
make -s -C $P
OBJS=$(ls $P/build/*.o $P/build/kernels/*.o | grep -v kernels/scan)
for v in "$@"; do
  IFS=x read R T M <<< "$v"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -DMDHB_SCAN_ROUNDS=$R -DMDHB_SCAN_THREADS=$T -DMDHB_SCAN_MINB=$M \
    -x cu -c $P/csrc/kernels/scan.cu -o build/scan_$v.o &
done
wait
for v in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/lib_scan_$v.so $OBJS build/scan_$v.o -ldl -lpthread
done
