#!/bin/sh
# A/B of the first-occurrence guard/bitmap probe cache operator (in-tree .cg vs ab/probe_ca .ca;
# build: sh tools/build_variant.sh probe_ca '-DFH_PROBE_CACHE=\"ca\"')
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for r in 1 2; do
 for L in paper_2306_10410_b200/libboba_b200.so ab/probe_ca/pkg/libboba_b200.so; do
  BOBA_LIB_PATH=$PWD/$L timeout 600 python tools/phase_ab.py c4,c5,c3,c2 10 2>&1 | grep digest | sed "s@^@$L @"
 done
done > gpurun_out/ab_probe.log
