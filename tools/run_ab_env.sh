# A/B of an environment switch: A = "$1=0", B = "$1=1" (same library)
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1 --steps 10"
for v in A B A B; do
  if [ $v = A ]; then V=0; else V=1; fi
  env $1=$V timeout 300 python bench.py $ARGS $2 > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernels_ms_per_step_serialized'])" >> gpurun_out/ab.log
done
