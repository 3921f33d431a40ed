# A/B: abl/base.so (A) vs the in-tree library (B), 256-position headline, 2 rounds each
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1 --steps 10"
for v in A B A B; do
  if [ $v = A ]; then L=abl/base.so; else L=paper_2311_15566_b200/_lib/libspotkm.so; fi
  SPOTKM_LIB=$L timeout 300 python bench.py $ARGS $1 > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['kernels_ms_per_step_serialized'])" >> gpurun_out/ab.log
done
