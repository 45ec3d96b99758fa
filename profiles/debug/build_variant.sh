#!/bin/bash
# build a variant library with extra nvcc defines into build/variant/<name>/liblvsg.so
# usage: build_variant.sh NAME "-DFOO=1 ..."
set -e
name=$1; defs=$2
out=build/variant/$name; mkdir -p $out
objs=""
for f in paper_2411_16680_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC --expt-relaxed-constexpr -I include $defs -c $f -o $out/$b.cu.o &
  objs="$objs $out/$b.cu.o"
done
wait
for f in paper_2411_16680_b200/csrc/*.cpp; do
  b=$(basename $f .cpp)
  g++ -O2 -std=c++20 -fPIC -I include -I /usr/local/cuda/include -c $f -o $out/$b.o
  objs="$objs $out/$b.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/liblvsg.so $objs -lcudart_static -lrt -ldl -lpthread
echo $out/liblvsg.so
