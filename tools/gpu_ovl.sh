#!/bin/bash
# C1 concurrent auxiliary grid (packer + filler on the idle SMs) A/B: parity tests of the
# new default, then the bench line per (SKB_RNN_XOVL, SKB_RNN_FOVL), then a launch list.
mkdir -p gpurun_out
SKB_RNN_XOVL=1 SKB_RNN_FOVL=1 timeout 120 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/ovl_b_first.json 2> gpurun_out/ovl_b_first.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/ovl_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ovl_parity.log
for xo in 0 1; do for fo in 0 1; do
  SKB_RNN_XOVL=$xo SKB_RNN_FOVL=$fo timeout 200 python bench.py --no-e2e --no-cpu > gpurun_out/ovl_b_${xo}${fo}.json 2> gpurun_out/ovl_b_${xo}${fo}.err
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ovl_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
