#!/bin/bash
# Builds probe variants of the tensor-core conv (LVSG_CONV_PROBE=k, see
# csrc/conv_tc.cu) as probe_libs/liblvsg_p<k>.so for profiles/conv_probe.py.
set -e
cd "$(dirname "$0")/.."
python paper_2411_16680_b200/build.py > /dev/null
mkdir -p build/probe probe_libs
objs=$(ls build/obj/*.o | grep -v conv_tc.cu.o)
for k in "$@"; do
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
     --expt-relaxed-constexpr -Iinclude -DLVSG_CONV_PROBE=$k \
     -c paper_2411_16680_b200/csrc/conv_tc.cu -o build/probe/conv_tc_$k.o &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o probe_libs/liblvsg_p$k.so $objs \
     build/probe/conv_tc_$k.o -lcudart_static -lrt -ldl -lpthread) &
done
wait
