# Closing check on the final code: every GPU test file (own timeout each), smoke, the
# default bench line and the reference arm
for f in test_daemon_gpu test_range_gpu test_estimator_gpu test_edge_gpu test_mapping_gpu test_sweep_gpu test_reshard_gpu test_k1_gpu test_reference_suite test_bench_contract_gpu test_reshard_multigpu; do
  echo "=== $f" >> gpurun_out/closing_tests.log
  timeout 600 python -m pytest tests/$f.py -q -m gpu -p no:cacheprovider >> gpurun_out/closing_tests.log 2>&1
  echo "EXIT $?" >> gpurun_out/closing_tests.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/closing_smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/closing_smoke.log
timeout 1500 python bench.py > gpurun_out/closing_bench.json 2> gpurun_out/closing_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/closing_bench_ref.json 2>> gpurun_out/closing_bench.err
