# end-of-session numbers: the four bench lines, DRAM traffic of one eager step
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final_resnet50.json 2> gpurun_out/final_resnet50.err
for c in resnet18 lenet mlp; do
  timeout 600 python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_traffic.log 2>&1
for c in resnet50 resnet18 lenet mlp; do cut -c1-260 gpurun_out/final_$c.json; done
