#!/bin/bash
# A/B the current build against ab/liblcae_*.so on the default bench (c3): prints kernel ms per variant.
# usage: tools/ab.sh [reps]
reps=${1:-2}
for i in $(seq $reps); do
  for lib in ab/liblcae_*.so ""; do
    name=${lib:-current}
    LCAE_LIB=${lib:+$PWD/$lib} python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
  done
done
