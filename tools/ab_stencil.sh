#!/bin/bash
# A/B the stencil micro-benchmark across alternative builds: tools/ab_stencil.sh SIZES lib1 lib2 ...
sizes=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$(basename $lib) rep$rep "
    EMHD_LIB=$lib python tools/bench_stencil.py $sizes | python -c "import json,sys; d=json.load(sys.stdin); print(' '.join('%s%d:%.1f'%(r['kind'],r['n'],r['us']) for r in d['results']))"
  done
done
