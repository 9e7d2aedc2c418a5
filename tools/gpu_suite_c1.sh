#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c1_rows.json 2> gpurun_out/bench_c1_rows.err
SKB_H2D_ROWS=0 timeout 600 python bench.py --no-cpu > gpurun_out/bench_c1_norows.json 2>> gpurun_out/bench_c1_rows.err
