set -e
ncu --set full --import-source on --clock-control none -k regex:"k_outer|k_fuse|k_sweep_expand" -c 12 -o gpurun_out/full_S4096 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-all-sizes > gpurun_out/ncu_full.log 2>&1
