#!/bin/bash
# usage: mkab.sh name "-Dflags..."
cd /root/repo/paper_2104_05877_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c csrc/sketch.cu -o /tmp/sketch_$1.o || exit 1
objs=$(ls build/*.o | grep -v '/sketch.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../ab/libskel_$1.so $objs /tmp/sketch_$1.o -lcudart -ldl
