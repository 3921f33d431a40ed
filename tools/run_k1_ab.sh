# K1 A/B: abl/base.so (A) vs the in-tree library (B), tools/k1_probe.py, 2 rounds each
for v in A B A B; do
  if [ $v = A ]; then L=abl/base.so; else L=paper_2311_15566_b200/_lib/libspotkm.so; fi
  echo -n "$v " >> gpurun_out/k1ab.log
  SPOTKM_LIB=$L timeout 300 python tools/k1_probe.py 2>> gpurun_out/k1ab.err | tail -1 >> gpurun_out/k1ab.log
done
