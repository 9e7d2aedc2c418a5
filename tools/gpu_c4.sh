#!/bin/bash
# C4 (L-BFGS, vector-stream tier): bench line + launch list + one full ncu capture.
mkdir -p gpurun_out
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c4 --impl reference --steps 1 --warmup 0 > gpurun_out/bench_c4_ref.json 2>> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 \
    -o gpurun_out/prof_stream -f python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --n 2000000 > gpurun_out/ncu_c4_full.log 2>&1
cat gpurun_out/bench_c4.json gpurun_out/bench_c4_ref.json; tail -3 gpurun_out/bench_c4.err
