#!/bin/sh
# usage: sh tools/ab_lib.sh NAME CFGS LIB_A LIB_B [TESTS] -- parity tests on the in-tree build, then
# per-phase times of two library builds interleaved twice (gpurun_out/ab_NAME.log)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
if [ -n "$5" ]; then
  timeout 1500 python -m pytest $5 -x -q > gpurun_out/parity_$1.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/parity_$1.log)"
fi
for r in 1 2; do
  for L in $3 $4; do
    BOBA_LIB_PATH=$PWD/$L timeout 900 python tools/phase_ab.py $2 10 2>&1 | grep digest | sed "s@^@$L @"
  done
done > gpurun_out/ab_$1.log
cat gpurun_out/ab_$1.log | cut -c1-220
