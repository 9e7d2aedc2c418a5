#!/bin/bash
# C2 backward: 4-way split-K over a 4-CTA cluster (SKB_TC_BWD_KS=4) vs 2-way
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -p no:cacheprovider > gpurun_out/c2_test.log 2>&1; echo "rc=$?" >> gpurun_out/c2_test.log
timeout 200 python tools/trace_c2.py > gpurun_out/c2_trace_ks4.txt 2>&1
timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_ks4.json 2> gpurun_out/c2ks4.err
SKB_TC_BWD_KS=2 timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_ks2.json 2>> gpurun_out/c2ks4.err
