#!/bin/bash
# C2 with the DSMEM split-K exchange: parity, trace, bench, launch list
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_train.py -x -q -p no:cacheprovider > gpurun_out/c2_test.log 2>&1; echo "rc=$?" >> gpurun_out/c2_test.log
timeout 200 python tools/trace_c2.py > gpurun_out/c2_trace.txt 2>&1
timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2.json 2>> gpurun_out/c2dsm.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
