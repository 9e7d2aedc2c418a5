#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiFwd -s 1 -c 1 -o gpurun_out/prof_c2fwd2 -f \
   python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c2fwd2.log 2>&1
