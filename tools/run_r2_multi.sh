# N-GPU legs: bench (mapping sweep plan-sharded + the context reshard), the
# multi-rank executor check, and NVLink counters for the copy kernel
N=${1:-2}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --steps 5 --warmup 3 --no-all-sizes > gpurun_out/bench_r2_${N}gpu.json 2> gpurun_out/bench_r2_${N}gpu.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 tools/reshard_check.py > gpurun_out/reshard_check_${N}gpu.log 2>&1
echo "EXIT $?" >> gpurun_out/reshard_check_${N}gpu.log
for m in pull push; do
  timeout 120 python tools/nvlink_probe.py $m 7.2 > gpurun_out/nvlink_probe_${m}.log 2>&1
  timeout 600 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum -k regex:k_copy --csv --log-file gpurun_out/r2_nvlink_${m}.csv python tools/nvlink_probe.py $m 7.2 > gpurun_out/ncu_nvlink_${m}.log 2>&1
done
