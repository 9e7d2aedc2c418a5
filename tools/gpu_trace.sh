mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "bench_path or full_size or widths or gru" > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
SKB_LIB_PATH=$PWD/paper_1810_08061_b200/libskb_trace.so timeout 120 python tools/trace_pair.py > gpurun_out/trace_pair.txt 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
