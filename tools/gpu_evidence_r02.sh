#!/bin/bash
# Round-2 evidence on one B200: smoke, full GPU suite, bench lines of every config (both
# arms), launch lists and one `ncu --set full` capture of each config's dominant kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c4 c5 c5m; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  timeout 600 python bench.py --config $c --impl reference --steps 2 --warmup 0 > gpurun_out/bench_${c}_ref.json 2>> gpurun_out/bench_$c.err
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file gpurun_out/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
for c in c2 c3 c4 c5 c5m; do
  timeout 900 ncu $M --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:rnn_fwd -s 1 -c 1 -o gpurun_out/prof_rnn -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 1200 ncu $F --kernel-name-base demangled -k regex:EpiBwd -s 1 -c 1 -o gpurun_out/prof_c2bwd -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 1200 ncu $F --kernel-name-base demangled -k regex:EpiFwd -s 1 -c 1 -o gpurun_out/prof_c2fwd -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu $F -k regex:stream_kernel -c 1 -o gpurun_out/prof_stream -f python tools/stream_micro_one.py micro_axpy 10000000 20 > /dev/null 2>&1
timeout 900 ncu $F -k regex:beam_rows -s 3 -c 1 -o gpurun_out/prof_beam_rows -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu $F -k regex:tree_cell -s 3 -c 1 -o gpurun_out/prof_tree_cell -f python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu $F -k regex:maml_task -s 1 -c 1 -o gpurun_out/prof_maml -f python bench.py --config c5m --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la gpurun_out; tail -3 gpurun_out/pytest_gpu.log
