#!/bin/bash
# build.sh NAME "-Dflags..."  : stream.cu with flags + the other current objects
set -e
cd /root/repo; python -m paper_2112_02052_b200._build >/dev/null
d=scratch/variants/$1; mkdir -p $d
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -O3 $2 -Xptxas -v -c paper_2112_02052_b200/csrc/${3:-stream}.cu -o $d/${3:-stream}.o 2> $d/ptxas.txt
objs=$(ls paper_2112_02052_b200/build/*.o | grep -v "/${3:-stream}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libtcg_b200.so $d/${3:-stream}.o $objs
true
