#!/bin/sh
# usage: sh tools/csr_ab_libs.sh CFGS REPS LIB... -- csr_ab.py per library build, interleaved twice
cfgs=$1; reps=$2; shift 2
for r in 1 2; do for lib in "$@"; do
  echo "== $lib"; BOBA_LIB_PATH=$lib python tools/csr_ab.py $cfgs $reps 2>&1 | grep median
done; done
