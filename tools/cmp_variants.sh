# usage: bash tools/cmp_variants.sh "a x ..."  -- parity subset + bench per BOBA_RADIX_CFG variant
VARS=${1:-"a m"}
for v in $VARS; do BOBA_RADIX_CFG=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rmat_pipeline or stability or radix_pass or tails" 2>&1 | tail -1; done
for v in $VARS $VARS; do BOBA_RADIX_CFG=$v python bench.py --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['roofline']['phases'].items()})"; done
