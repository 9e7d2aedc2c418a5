#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiLogits -s 4 -c 1 -o gpurun_out/prof_c3log -f \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c3log.log 2>&1
