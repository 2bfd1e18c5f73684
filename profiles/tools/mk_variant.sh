#!/bin/bash
# usage: abvar/mk.sh NAME "flags"  -> abvar/NAME.so
cd /root/repo/paper_2507_04991_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xptxas -O3 -I../../include $2 dg_kernels.cu host.cpp -o /root/repo/abvar/$1.so -lcudart -lnccl
