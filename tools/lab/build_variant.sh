#!/bin/bash
# build a variant of libalyab200.so with extra -D flags: tools/lab/build_variant.sh NAME -DFOO=1 ...
name=$1; shift
srcs=$(python -c "from paper_2005_05899_b200 import build; print(' '.join(str(build.CSRC / s) for s in build.SOURCES))")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr "$@" -I include -o tools/lab/lib_$name.so $srcs
