#!/bin/bash
# Round-end evidence on one B200: full GPU test suite, bench lines of every
# config, launch lists and one full ncu capture of each config's own dominant kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in c1 c2 c3 c4 c5 c5m; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  timeout 600 python bench.py --config $c --impl reference --steps 2 --warmup 0 > gpurun_out/bench_${c}_ref.json 2>> gpurun_out/bench_$c.err
done
# launch lists (cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5m.csv python bench.py --config c5m --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
# full captures of our own dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rnn_fwd -s 1 -c 1 -o gpurun_out/prof_rnn -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 -o gpurun_out/prof_stream -f python tools/stream_micro_one.py micro_axpy 10000000 20 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_rows -s 3 -c 1 -o gpurun_out/prof_beam_rows -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lstm_bwd_cell -s 5 -c 1 -o gpurun_out/prof_train_cell -f python bench.py --config c2 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_cell -s 3 -c 1 -o gpurun_out/prof_tree_cell -f python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maml_task -s 1 -c 1 -o gpurun_out/prof_maml -f python bench.py --config c5m --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la gpurun_out; tail -3 gpurun_out/pytest_gpu.log
