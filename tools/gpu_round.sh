#!/bin/sh
# sharded tests (incl. the NCCL C-ABI entry), racecheck after the dynamic-set fix, the full bench pair
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_host_io.py -x -q 2>&1 | tail -5
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/sanitize_racecheck.log | tail -1)"
s=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - s ))"
s=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))"
