#!/bin/bash
# Launch list + one full ncu capture of the persistent recurrent kernel (1 GPU).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rnn_fwd -s 1 -c 1 \
    -o gpurun_out/prof_rnn -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:pack_x -s 1 -c 1 \
    -o gpurun_out/prof_pack -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_pack.log 2>&1
ls -la gpurun_out
