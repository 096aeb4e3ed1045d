#!/bin/sh
# ncu --set full of one launch of each c4 hot kernel (tools/profile_step.py 26 1), report in gpurun_out/
K='regex:k_radix_downsweep|k_relabel_range|k_first_hit_static|k_assign|k_spmv_merge|k_radix_upsweep|k_mark'
ncu --set full --clock-control none --import-source on -k "$K" --launch-count 12 -o gpurun_out/r02_c4_full python tools/profile_step.py 26 1 > gpurun_out/r02_c4_full.log 2>&1
echo "ncu rc=$?"
