#!/bin/bash
# C2 evidence refresh: bench (both arms), launch list, ncu --set full of both step kernels, trace
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c2 --impl reference --steps 2 --warmup 0 > gpurun_out/bench_c2_ref.json 2>> gpurun_out/bench_c2.err
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 900 ncu $M --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 1200 ncu $F --kernel-name-base demangled -k regex:EpiBwd -s 1 -c 1 -o gpurun_out/prof_c2bwd -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 1200 ncu $F --kernel-name-base demangled -k regex:EpiFwd -s 1 -c 1 -o gpurun_out/prof_c2fwd -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 200 python tools/trace_c2.py > gpurun_out/c2_trace.txt 2>&1
