# end-of-session verification: GPU tests, smoke, the four bench lines, the launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final_resnet50.json 2> gpurun_out/final_resnet50.err
for c in resnet18 lenet mlp; do
  timeout 600 python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/conv_bench.py --stats > gpurun_out/conv_final.txt 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for c in resnet50 resnet18 lenet mlp reference; do cut -c1-200 gpurun_out/final_$c.json; done
tail -1 gpurun_out/conv_final.txt
