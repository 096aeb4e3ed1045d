#!/bin/sh
# A/B of the rank-assignment batch size (needs: sh tools/build_variant.sh base "" built from the one-at-a-time
# source, b8 "-DASSIGN_BATCH=8", b2 "-DASSIGN_BATCH=2"); the in-tree build is batch 4 at the time of the run.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for r in 1 2; do
 for L in ab/base/pkg/libboba_b200.so paper_2306_10410_b200/libboba_b200.so ab/b8/pkg/libboba_b200.so ab/b2/pkg/libboba_b200.so; do
  BOBA_LIB_PATH=$PWD/$L timeout 600 python tools/phase_ab.py c4,c5,c2 10 2>&1 | grep digest | sed "s@^@$L @"
 done
done > gpurun_out/ab_assign.log
timeout 1200 python -m pytest tests/test_gpu_baseline_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/parity_assign.log 2>&1; echo parity rc=$?; tail -2 gpurun_out/parity_assign.log
