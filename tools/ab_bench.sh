#!/bin/bash
# A/B timing of library variants on the GPU box (dev tool): bench.py per variant,
# one JSON summary line each into gpurun_out/ab.log.
cd "$(dirname "$0")/.."
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset GRASP_LIB; else export GRASP_LIB=$PWD/paper_2412_16490_b200/_lib/variants/libgrasp_b200_$lib.so; fi
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ab_$lib.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$lib.json').read().strip().splitlines()[-1])
o = d['roofline'].get('ops', {}); q = max(1, o.get('point_queries', 1))
print('$lib', d['value'], {k: round(v,1) for k,v in d['roofline']['kernel_ms'].items()},
      {k: round(o.get(k, 0) / q, 2) for k in ('plane_tests', 'triangle_tests')})" >> gpurun_out/ab.log
done
