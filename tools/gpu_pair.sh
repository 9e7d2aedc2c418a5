mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
SKB_RNN_PAIR=0 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
