#!/bin/bash
# C5 TreeLSTM: engine path (default) vs cuBLAS level GEMMs
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tree.py -x -q -p no:cacheprovider > gpurun_out/tree_test.log 2>&1; echo "rc=$?" >> gpurun_out/tree_test.log
timeout 300 python bench.py --config c5 --no-cpu > gpurun_out/bench_c5_engine.json 2> gpurun_out/tree.err
SKB_TREE_TC=1 timeout 300 python bench.py --config c5 --no-cpu > gpurun_out/bench_c5_tc.json 2>> gpurun_out/tree.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c5_engine.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
