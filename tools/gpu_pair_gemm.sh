#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/gemm_test.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_test.log
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe.txt 2>&1
