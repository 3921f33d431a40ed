python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for g in 1 12 30; do SK_OUTER_GMIN=$g python tools/sweep_classes.py 256 4096 > gpurun_out/cls_g$g.json 2>&1; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-all-sizes > gpurun_out/b1.json 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-sizes --positions 1024 --sets 512 > gpurun_out/b2.json 2>&1
SK_OUTER_GMIN=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-sizes --positions 1024 --sets 512 > gpurun_out/b3.json 2>&1
