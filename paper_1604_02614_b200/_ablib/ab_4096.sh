for lib in "" "EMHD_LIB=paper_1604_02614_b200/_ablib/libemhd_nraw1.so"; do
  for n in 4096 2048 1024; do
    echo "== $lib n=$n"
    env $lib python bench.py --n $n --steps 2 --warmup 1 --jv 5 --no-two-pass --no-secondary --no-cpu-baseline --no-trajectory --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%.1f it/s' % d['value'], 'iter_frac %.3f' % d['iteration_roofline']['frac'], 'sp', d['iteration_roofline']['second_pass_iterations'], ' '.join('%s:%.1fus/%.2f' % (k['kernel'].replace('emhd_',''), k['avg_us'], k['frac']) for k in d['kernels'][:5]))"
  done
done
