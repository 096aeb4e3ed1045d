#!/bin/sh
# usage: sh tools/ab_multi.sh NAME CFGS LIB... -- per-phase times of several library builds, interleaved twice
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
name=$1; cfgs=$2; shift 2
for r in 1 2; do
  for L in "$@"; do
    BOBA_LIB_PATH=$PWD/$L timeout 900 python tools/phase_ab.py $cfgs 10 2>&1 | grep digest | sed "s@^@$L @"
  done
done > gpurun_out/ab_$name.log
cat gpurun_out/ab_$name.log
