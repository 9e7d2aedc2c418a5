#!/bin/bash
# C2 forward: CTA-pair tiles with 2-way interleaved split-K over a 4-CTA cluster (SKB_TC_FWD_KS=2)
mkdir -p gpurun_out
SKB_TC_FWD_KS=2 timeout 600 python -m pytest tests/test_gpu_train.py -x -q -p no:cacheprovider -k "oracle" > gpurun_out/c2_test.log 2>&1; echo "rc=$?" >> gpurun_out/c2_test.log
SKB_TC_FWD_KS=2 timeout 200 python tools/trace_c2.py > gpurun_out/c2_trace_fks.txt 2>&1
SKB_TC_FWD_KS=2 timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_fks2.json 2> gpurun_out/c2fks.err
timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_fks1.json 2>> gpurun_out/c2fks.err
