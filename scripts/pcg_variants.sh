#!/bin/bash
# fat-thread PCG builds on the throughput workloads:  scripts/pcg_variants.sh  (run on the GPU box)
for w in c3 c5; do
  for minb in 0 1 2; do
    printf "%s GATO_PCG_MINB=%s  " $w $minb
    GATO_PCG_MINB=$minb python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms_per_step']
print('step %.3f ms  pcg %.3f  schur %.3f lin %.3f ls %.3f  its %.1f' % (d['ms_per_step'], k['pcg'], k['schur'], k['linearize'], k['linesearch'], d['pcg_iterations_mean']))"
  done
done
