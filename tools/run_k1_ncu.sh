# ncu --set full of K1 (k_weights) from tools/k1_probe.py, summarised on the box
R=/tmp/ncu_k1; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_weights -c 2 -o $R/k1 python tools/k1_probe.py > gpurun_out/ncu_k1.log 2>&1
python tools/ncu_summary.py $R/k1.ncu-rep --stalls > gpurun_out/r2_ncu_k1.txt 2>&1
python tools/ncu_lines.py $R/k1.ncu-rep k_weights 25 > gpurun_out/r2_lines_k1.txt 2>&1
ncu -i $R/k1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/r2_ncu_k1_dram.csv 2>&1
