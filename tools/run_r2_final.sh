# Final validation on one GPU: every GPU test file (own timeout each), smoke,
# the default bench line + the reference arm, the launch list, ncu captures
# summarised on the box, the K1 probe.
for f in test_daemon_gpu test_range_gpu test_estimator_gpu test_edge_gpu test_mapping_gpu test_sweep_gpu test_reshard_gpu test_k1_gpu test_reference_suite test_bench_contract_gpu test_reshard_multigpu; do
  echo "=== $f" >> gpurun_out/final_tests.log
  timeout 600 python -m pytest tests/$f.py -q -m gpu -p no:cacheprovider >> gpurun_out/final_tests.log 2>&1
  echo "EXIT $?" >> gpurun_out/final_tests.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/final_smoke.log
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2>> gpurun_out/final_bench.err
ARGS="--no-all-sizes --no-cpu-baseline --no-dropin --no-k1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_N256.csv python bench.py --steps 2 --warmup 3 $ARGS > /dev/null 2>&1
bash tools/run_r2_ncu.sh > gpurun_out/run_ncu.log 2>&1
timeout 300 python tools/k1_probe.py > gpurun_out/final_k1.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_weights --csv --log-file gpurun_out/final_k1_dram.csv python tools/k1_probe.py > /dev/null 2>&1
