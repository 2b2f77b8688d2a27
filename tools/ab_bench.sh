#!/bin/bash
# A/B timing of library builds on the headline + mid sizes: tools/ab_bench.sh build/libA.so build/libB.so ...
for lib in "$@"; do
  for cfg in "config4" "config3" "config2"; do
    MLA_B200_LIB=$PWD/$lib python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --config $cfg 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$lib', d['config']['workload'], d['ms_per_step'], 'ms', d['value'], 'GFLOP/s')"
  done
done
