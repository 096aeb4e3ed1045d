#!/bin/sh
# Range-pass relabel at n = 2^24 (c5, c3; BOBA_RL_PASSES forces it) against the single pass
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for r in 1 2; do
  for v in "X=1" "BOBA_RL_PASSES=2" "BOBA_RL_PASSES=3" "BOBA_RL_PASSES=4"; do
    env $v timeout 600 python tools/phase_ab.py c5,c3 10 2>&1 | grep digest | sed "s/^/[$v] /"
  done
done > gpurun_out/ab_rlpasses.log
cat gpurun_out/ab_rlpasses.log
