#!/bin/bash
# C2 after the residency checks: tests, bench, and which step kernels ran
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -p no:cacheprovider > gpurun_out/c2_test.log 2>&1; echo "rc=$?" >> gpurun_out/c2_test.log
timeout 200 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2_fit.json 2> gpurun_out/c2fit.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_fit.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
