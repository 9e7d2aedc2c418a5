#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py -q -p no:cacheprovider > gpurun_out/c3_test.log 2>&1; echo "rc=$?" >> gpurun_out/c3_test.log
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
SKB_DEC_CUBLAS=1 timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/bench_c3_cublas.json 2>> gpurun_out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
