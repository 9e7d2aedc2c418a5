#!/bin/bash
mkdir -p gpurun_out
for ch in 12 24 36; do
  SKB_PIPELINE_CHUNKS=$ch timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/e2e_ch$ch.json 2>> gpurun_out/e2e.err
done
