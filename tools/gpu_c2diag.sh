#!/bin/bash
mkdir -p gpurun_out
for dg in 0 1 2 3; do
  SKB_TRAIN_PDL=0 SKB_TC_DIAG=$dg timeout 300 python bench.py --config c2 --no-cpu --steps 3 > gpurun_out/c2diag_$dg.json 2>> gpurun_out/c2diag.err
done
timeout 300 python tools/gemm_step_probe.py > gpurun_out/step_probe.txt 2>&1
