# ncu --set full of the coded k_fuse launches of one 256-position pass, summarised on the box
R=/tmp/ncu_fc; mkdir -p $R
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fuse|k_outer" -c 12 -o $R/fc python bench.py --steps 1 --warmup 1 $ARGS > gpurun_out/ncu_fc.log 2>&1
python tools/ncu_summary.py $R/fc.ncu-rep --stalls > gpurun_out/ncu_fc_summary.txt 2>&1
python tools/ncu_lines.py $R/fc.ncu-rep k_fuse 40 > gpurun_out/ncu_fc_lines.txt 2>&1
python tools/ncu_lines.py $R/fc.ncu-rep k_outer 30 > gpurun_out/ncu_fc_lines_outer.txt 2>&1
