#!/bin/bash
# dev: kernel time of the default bench under each LCAE_DEBUG_FLAGS value (work-skipping ceilings; numbers only)
for fl in ${@:-0 1 2 3}; do
  LCAE_DEBUG_FLAGS=$fl python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flags=$fl', round(d['roofline']['kernel_ms'],3))"
done
