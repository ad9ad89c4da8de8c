# launch list + DRAM traffic of one ResNet-50 step, per-layer conv table, GEMM ncu summary
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_traffic.log 2>&1
timeout 300 python tools/conv_bench.py > gpurun_out/conv_bench.txt 2>&1
timeout 300 python tools/bn_bench.py > gpurun_out/bn_bench.txt 2>&1
ncu --set full --clock-control none -k regex:k_tc_gemm -c 12 -o /tmp/gemm_full python tools/conv_bench.py --once --layers 2,3,4,16 > /dev/null 2>&1
ncu -i /tmp/gemm_full.ncu-rep --page details --csv > gpurun_out/gemm_full_details.csv
ncu -i /tmp/gemm_full.ncu-rep --page raw --csv > gpurun_out/gemm_full_raw.csv
tail -1 gpurun_out/conv_bench.txt
