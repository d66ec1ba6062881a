#!/bin/bash
# A/B variant of the library: one source (default rr_trace.cu) recompiled
# with extra defines, linked with the other objects of the current build.
#   bash profiles/ab_build.sh <name> "-DFOO=1 -DBAR" [rr_sah]   -> build/ab/<name>/libroomray_b200.so
# time variants with: python profiles/ab_time.py c5 build/ab/a/libroomray_b200.so build/ab/b/...
set -e
cd "$(dirname "$0")/.."
make -s -C paper_1811_05784_b200/csrc ../libroomray_b200.so
mkdir -p build/ab/$1
cd paper_1811_05784_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-O2 \
     -I../../include $2 -c ${3:-rr_trace}.cu -o ../../build/ab/$1/${3:-rr_trace}.o
objs=$(ls ../../build/*.o | grep -v "/${3:-rr_trace}.o\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/ab/$1/libroomray_b200.so $objs \
     ../../build/ab/$1/${3:-rr_trace}.o -lnccl
