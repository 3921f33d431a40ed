python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
SPOTKM_LIB=altlib/base.so python tools/sweep_classes.py 256 4096 > gpurun_out/clsA.json 2>&1
python tools/sweep_classes.py 256 4096 > gpurun_out/clsB.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-all-sizes > gpurun_out/b1.json 2>&1
