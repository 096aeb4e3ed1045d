#!/bin/sh
# Round-end evidence on the final code: sanitizers, per-phase DRAM bytes, launch list, the bench pair.
sh tools/sanitize.sh
sh tools/gpu_traffic.sh
sh tools/run_bench_pair.sh 20 5
