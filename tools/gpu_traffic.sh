#!/bin/sh
# per-phase DRAM bytes (one direct step) for every BASELINE config; launch list of a bench step
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for a in "22 c2" "grid c3" "24 c5" "26 c4"; do
  set -- $a
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/tr_$2.csv python tools/profile_step.py $1 1 > /dev/null 2>&1
  python tools/traffic_csv.py gpurun_out/tr_$2.csv $2 > gpurun_out/traffic_$2.json; echo "$2 rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --quick --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1; echo "launches rc=$?"
python -m pytest tests/test_gpu_host_io.py -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"; tail -n 3 gpurun_out/bench_quick.err
