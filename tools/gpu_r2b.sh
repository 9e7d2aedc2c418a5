mkdir -p gpurun_out
timeout 120 python tools/umma_pair.py > gpurun_out/umma_pair.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
