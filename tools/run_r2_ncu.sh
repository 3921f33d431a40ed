# ncu captures summarised ON the box (reports themselves stay in /tmp: too big to ship back)
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1"
R=/tmp/ncu_r2; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_outer|k_fuse|k_sweep|k_overflow" -c 24 -o $R/full_N256 python bench.py --steps 1 --warmup 1 $ARGS > gpurun_out/ncu_f256.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_outer|k_fuse|k_overflow" -c 16 -o $R/full_N1024 python bench.py --positions 1024 --sets 256 --steps 1 --warmup 1 $ARGS > gpurun_out/ncu_f1024.log 2>&1
for N in 256 1024; do
  python tools/ncu_summary.py $R/full_N$N.ncu-rep --stalls > gpurun_out/r2_ncu_full_N$N.txt 2>&1
  python tools/ncu_lines.py $R/full_N$N.ncu-rep k_outer 30 > gpurun_out/r2_lines_k_outer_N$N.txt 2>&1
  python tools/ncu_lines.py $R/full_N$N.ncu-rep k_fuse 30 > gpurun_out/r2_lines_k_fuse_N$N.txt 2>&1
  python tools/ncu_to_json.py $R/full_N$N.ncu-rep gpt-20b-N$N-S$([ $N = 256 ] && echo 4096 || echo 256) > gpurun_out/r2_ncu_json_N$N.log 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_r2.json
