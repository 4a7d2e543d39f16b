#!/bin/bash
# debug build of libsv with globaltimer instrumentation (-DSV_TRACE) -> libsv_trace.so
cd "$(dirname "$0")/.." && mkdir -p /tmp/trb
for f in paper_2509_24328_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -DSV_TRACE -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I include -c $f -o /tmp/trb/$(basename $f .cu).o || exit 1
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared /tmp/trb/*.o -o paper_2509_24328_b200/libsv_trace.so -cudart static
