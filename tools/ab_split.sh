#!/bin/sh
# Rank assignment split (upper vertices on a side stream beside the first relabel range pass):
# parity, then direct-call phase times and the captured bench step, with and without it.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -x -q > gpurun_out/parity_split.log 2>&1
echo "parity rc=$? $(tail -1 gpurun_out/parity_split.log)"
for r in 1 2; do
  BOBA_NO_ASSIGN_SPLIT=1 timeout 600 python tools/phase_ab.py c4 10 2>&1 | grep digest | sed 's/^/nosplit /'
  timeout 600 python tools/phase_ab.py c4 10 2>&1 | grep digest | sed 's/^/split   /'
done > gpurun_out/ab_split.log
BENCH_ARGS="--quick" bash tools/ab.sh "BOBA_NO_ASSIGN_SPLIT=1" "BOBA_SPLIT=default" >> gpurun_out/ab_split.log 2>&1
cat gpurun_out/ab_split.log
