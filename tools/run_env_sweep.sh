# one environment knob over several values: tools/run_env_sweep.sh VAR "v1 v2 ..." "bench args"
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1 --steps 4 $3"
for r in 1 2; do for V in $2; do
  env $1=$V timeout 400 python bench.py $ARGS > gpurun_out/sw_$V.json 2>> gpurun_out/sw.err
  python -c "import json;d=json.loads(open('gpurun_out/sw_$V.json').read().splitlines()[-1]);print('$1=$V', round(d['value']), d['ms_per_step'], {k: round(v,2) for k, v in d['kernels_ms_per_step_serialized'].items()})" >> gpurun_out/sw.log
done; done
