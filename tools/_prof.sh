set -e
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-all-sizes > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_outer|k_fuse|k_sweep_expand" -c 12 -o gpurun_out/full_S4096 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-all-sizes > gpurun_out/ncu_full.log 2>&1
