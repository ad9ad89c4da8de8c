# one build->measure iteration: GPU tests, selected conv layers, bench line,
# ncu --set full of the selected forward GEMMs (the stem and the 64-channel 3x3)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/conv_bench.py --stats --layers ${LAYERS:-0,2,6,10} > gpurun_out/conv_sel.txt 2>&1
timeout 500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -c 3 -o /tmp/sel_full python tools/conv_bench.py --once --stats --layers 0,2 --passes fwd > gpurun_out/ncu_sel.log 2>&1
cp /tmp/sel_full.ncu-rep gpurun_out/ 2>/dev/null
fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/conv_sel.txt; cat gpurun_out/bench.json | cut -c1-400
