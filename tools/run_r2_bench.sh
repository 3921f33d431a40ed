set -x
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1"
for v in A B A B; do
  if [ $v = A ]; then L=abl/base.so; else L=paper_2311_15566_b200/_lib/libspotkm.so; fi
  SPOTKM_LIB=$L timeout 300 python bench.py $ARGS --steps 10 > gpurun_out/ab2_$v.json 2>> gpurun_out/ab2.err
  python -c "import json;d=json.loads(open('gpurun_out/ab2_$v.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['kernels_ms_per_step_serialized'])" >> gpurun_out/ab2.log
done
timeout 1500 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2c_ref.json 2>> gpurun_out/bench_r2c.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_N256.csv python bench.py --steps 2 --warmup 1 $ARGS > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_weights --csv --log-file gpurun_out/r2_k1.csv python tools/k1_probe.py > gpurun_out/k1_probe.log 2>&1
