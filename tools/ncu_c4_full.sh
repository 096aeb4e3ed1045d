#!/bin/sh
# ncu --set full of the first launch of each c4 hot kernel (tools/profile_step.py 26 1); reports in gpurun_out/
for k in k_radix_downsweep k_radix_upsweep k_relabel_range k_first_hit_static k_assign k_mark k_spmv_merge; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-count 1 -o gpurun_out/r02_c4_$k \
      python tools/profile_step.py 26 1 > gpurun_out/r02_c4_$k.log 2>&1
  echo "$k rc=$?"
done
