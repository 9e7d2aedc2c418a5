mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rnn_fwd_pair -s 2 -c 1 \
    -o gpurun_out/prof_pair -f python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_pair.log 2>&1
