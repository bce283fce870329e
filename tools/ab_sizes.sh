#!/bin/bash
# config-2 step (arnoldi m=40) at several grid sizes with the per-kernel table: bash tools/ab_sizes.sh
for n in 4096 2048 1024 512; do
  echo "== n=$n"
  python bench.py --n $n --steps 3 --warmup 2 --jv 5 --no-two-pass --no-secondary --no-cpu-baseline --no-trajectory --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%.1f it/s' % d['value'], 'iter_frac %.3f' % d['iteration_roofline']['frac'], 'sp', d['iteration_roofline']['second_pass_iterations'], ' '.join('%s:%.1fus/%.2f' % (k['kernel'].replace('emhd_',''), k['avg_us'], k['frac']) for k in d['kernels'][:4]))"
done
