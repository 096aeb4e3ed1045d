#!/bin/sh
# usage: sh tools/spmv_ab_libs.sh CFGS REPS LIB... -- spmv_lib_ab.py per library build, interleaved twice
cfgs=$1; reps=$2; shift 2
for r in 1 2; do for lib in "$@"; do
  BOBA_LIB_PATH=$lib python tools/spmv_lib_ab.py $cfgs $reps 2>&1 | grep -v Warn | sed "s|^|$(dirname $lib | cut -c1-20) |"
done; done
