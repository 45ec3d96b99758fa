#!/bin/bash
# Probe variants of the Winograd conv (LVSG_CONV_PROBE=k in csrc/conv_wino.cu).
set -e
cd "$(dirname "$0")/.."
python paper_2411_16680_b200/build.py > /dev/null
mkdir -p build/probe probe_libs
objs=$(ls build/obj/*.o | grep -v conv_wino.cu.o)
for k in "$@"; do
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
     --expt-relaxed-constexpr -Iinclude -DLVSG_CONV_PROBE=$k \
     -c paper_2411_16680_b200/csrc/conv_wino.cu -o build/probe/conv_wino_$k.o &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o probe_libs/liblvsg_w$k.so $objs \
     build/probe/conv_wino_$k.o -lcudart_static -lrt -ldl -lpthread) &
done
wait
