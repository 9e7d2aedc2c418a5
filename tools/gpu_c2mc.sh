#!/bin/bash
# C2 forward: A boxes multicast across two CTA pairs (SKB_TC_FWD_MC=1) vs one pair per cluster
mkdir -p gpurun_out
SKB_TC_FWD_MC=1 timeout 300 python -m pytest tests/test_gpu_train.py -x -q -p no:cacheprovider -k "oracle" > gpurun_out/c2_test.log 2>&1; echo "rc=$?" >> gpurun_out/c2_test.log
SKB_TC_FWD_MC=1 timeout 200 python tools/trace_c2.py > gpurun_out/c2_trace_mc.txt 2>&1
SKB_TC_FWD_MC=1 timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_mc.json 2> gpurun_out/c2mc.err
timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_nomc.json 2>> gpurun_out/c2mc.err
