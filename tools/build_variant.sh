#!/bin/bash
# build a libbingo variant with extra -D flags into build/variants/<name>/libbingo.so
name=$1; shift
d=build/variants/$name; mkdir -p $d
for f in paper_2504_10233_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I include -I paper_2504_10233_b200/csrc "$@" -c $f -o $d/$(basename $f .cu).o &
done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libbingo.so $d/*.o -lcudart
echo $d/libbingo.so
