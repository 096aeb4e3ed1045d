#!/bin/sh
# Relabel range passes with the label slice in the persisting L2 set-aside (BOBA_RL_PERSIST=1),
# 2 / 3 / 4 passes, against the default (2 passes, evict-last hints only); c4 per-phase times.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for r in 1 2; do
  for v in "X=1" "BOBA_RL_PERSIST=1" "BOBA_RL_PERSIST=1 BOBA_RL_PASSES=3" "BOBA_RL_PERSIST=1 BOBA_RL_PASSES=4"; do
    env $v timeout 600 python tools/phase_ab.py c4 10 2>&1 | grep digest | sed "s/^/[$v] /"
  done
done > gpurun_out/ab_persist.log
cat gpurun_out/ab_persist.log
