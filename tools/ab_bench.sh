#!/bin/bash
# A/B bench.py under environment variants: tools/ab_bench.sh "VAR=a" "VAR=b" ...  (extra bench args in BENCH_ARGS)
for rep in 1 2; do
  for v in "$@"; do
    echo -n "$v rep$rep "
    env $v python bench.py --no-cpu-baseline --no-e2e --no-trajectory $BENCH_ARGS 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%.1f it/s' % d['value'], ' '.join('%s:%.1fus/%.2f' % (k['kernel'].replace('emhd_',''), k['avg_us'], k['frac']) for k in d['kernels'][:4]))"
  done
done
