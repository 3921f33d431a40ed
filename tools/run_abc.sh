# A/B/C: abl/base.so, the in-tree library, abl/c.so
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1 --steps 10"
for v in A B C A B C; do
  case $v in A) L=abl/base.so;; B) L=paper_2311_15566_b200/_lib/libspotkm.so;; C) L=abl/c.so;; esac
  SPOTKM_LIB=$L timeout 300 python bench.py $ARGS $1 > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['kernels_ms_per_step_serialized'])" >> gpurun_out/ab.log
done
