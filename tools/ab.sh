# usage: bash tools/ab.sh "ENV1=a ENV2=b" "ENV3=c" ...  -- bench (no CPU leg) per env setting, twice interleaved
# extra bench args via BENCH_ARGS (e.g. BENCH_ARGS="--config c3")
for rep in 1 2; do
for v in "$@"; do env $v python bench.py --no-cpu --no-spmv-c3 --steps 20 $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['roofline']['phases'].items()}, 'spmv', (d.get('spmv',{}).get('c2') or d.get('spmv',{})).get('spmv_ms_boba'), (d.get('spmv',{}).get('c2') or d.get('spmv',{})).get('spmv_ms_random'))"; done
done
