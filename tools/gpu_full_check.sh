#!/bin/sh
# The driver's GPU checks: the -m gpu suite, smoke(), a short bench without the CPU legs.
python -m pytest tests -m gpu -x -q --durations=8 2>&1 | tail -25
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"; tail -n 3 gpurun_out/bench_quick.err
