#!/bin/bash
# build a variant of libalyab200.so with extra -D flags: tools/lab/build_variant.sh NAME -DFOO=1 ...
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr "$@" -I include -o tools/lab/lib_$name.so \
  paper_2005_05899_b200/csrc/{ab_api,ab_element,ab_solver,ab_node,ab_gradop,ab_cg_dd,ab_wall}.cu
