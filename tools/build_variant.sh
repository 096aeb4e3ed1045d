#!/bin/sh
# usage: sh tools/build_variant.sh NAME "-DMACRO=1 ..." -> ab/NAME/pkg/libboba_b200.so (for BOBA_LIB_PATH A/B runs)
set -e
d=ab/$1
rm -rf $d; mkdir -p $d/pkg
cp -r include $d/include
cp -r paper_2306_10410_b200/csrc $d/pkg/csrc
rm -rf $d/pkg/csrc/build
make -s -j8 -C $d/pkg/csrc NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2"
ls -la $d/pkg/libboba_b200.so
