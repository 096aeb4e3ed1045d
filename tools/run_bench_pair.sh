#!/bin/sh
# Both arms as the driver runs them (N = 1), wall time of each.
S=${1:-20}; W=${2:-5}
start=$(date +%s); python bench.py --gpus 1 --steps $S --warmup $W > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - start ))s"
start=$(date +%s); python bench.py --impl reference --gpus 1 --steps $S --warmup $W > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
