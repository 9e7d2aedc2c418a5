#!/bin/bash
# C1 e2e (host -> execute_many -> host) vs copy/compute pipeline depth
for c in ${CHUNKS:-4 8 16 32}; do
  SKB_PIPELINE_CHUNKS=$c python bench.py --steps 3 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.load(sys.stdin); print('chunks', $c, 'e2e', round(d['e2e']['value']), 'ms', round(d['e2e']['ms_per_step'],2))"
done
