for r in 1 2; do for L in altlib/ff1.so altlib/ff0.so altlib/ff7.so; do
  n=$(basename $L .so)
  SPOTKM_LIB=$L SK_PRECODED=0 timeout 300 python bench.py --no-all-sizes --no-cpu-baseline --no-dropin --no-k1 --steps 10 > gpurun_out/lib_$n.json 2>> gpurun_out/lib.err
  python -c "import json;d=json.loads(open('gpurun_out/lib_$n.json').read().splitlines()[-1]);print('$n', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k, v in d['kernels_ms_per_step_serialized'].items()})" >> gpurun_out/lib.log
done; done
