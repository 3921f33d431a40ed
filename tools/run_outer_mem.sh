# which k_outer source lines move the bytes: the k_outer<3,1,1> launch, source-level memory counters
R=/tmp/ncu_om; mkdir -p $R
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_outer" -s 2 -c 1 -o $R/om python bench.py --steps 1 --warmup 1 $ARGS > gpurun_out/ncu_om.log 2>&1
python tools/ncu_line_mem.py $R/om.ncu-rep k_outer 25 > gpurun_out/outer_mem_lines.txt 2>&1
