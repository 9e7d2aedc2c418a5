mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "bench_path or full_size or widths or gru" > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
for v in "X=0" "SKB_RNN_INFILL=1" "SKB_RNN_ACT=0"; do
  env $v timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.json').readline()); r=d['roofline']; print('$v', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'ms frac',round(r['frac'],3),'kernel',round(r['kernel_ms'],3))" >> gpurun_out/ab.txt 2>&1 || tail -2 gpurun_out/ab.err >> gpurun_out/ab.txt
done
