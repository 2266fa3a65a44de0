#!/bin/bash
# Build lib/libcpfit_gpu_stamps.so: the normal objects with als.cu compiled -DCPFIT_NORM_STAMPS
# (globaltimer stamps inside normalize_kernel, read by tools/norm_stamps.py). Run tools/mk.sh first.
set -e
cd "$(dirname "$0")/../paper_1105_5331_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -DCPFIT_NORM_STAMPS -c als.cu -o ../build/als_stamps.o
cd ../build
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libcpfit_gpu_stamps.so accel.o \
    als_stamps.o capi.o dense.o peaks.o poly.o problems.o solver.o sparse.o tensor.o -Xcompiler -fopenmp -lgomp
