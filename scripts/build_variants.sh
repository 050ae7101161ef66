#!/bin/bash
# Build libnef variants with different -D flags for kernels_tc.cu (diagnostics):
#   scripts/build_variants.sh tag1="-DX=1" tag2="-DX=2" ...  -> paper_2602_02759_b200/libnef_<tag>.so
set -e
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr"
make -s -j8 >/dev/null
for spec in "$@"; do
  tag=${spec%%=*}; defs=${spec#*=}
  ( $NVCC $FLAGS $defs -c paper_2602_02759_b200/csrc/kernels_tc.cu -o /tmp/ktc_$tag.o &&
    $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o paper_2602_02759_b200/libnef_$tag.so \
      build/obj/kernels_ffma.cu.o /tmp/ktc_$tag.o build/obj/api.cpp.o build/obj/plan.cpp.o -ldl ) &
done
wait
ls -la paper_2602_02759_b200/libnef_*.so
