# round-2 re-entry check: GPU tests, smoke, bench line, and full ncu captures of
# the stem fprop and the 64-channel 3x3 fprop (the two furthest from their bounds)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/smoke.log 2>&1
timeout 500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/conv_bench.py --stats --layers 0,2,6,10 > gpurun_out/conv_sel.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -c 3 -o /tmp/sel_full python tools/conv_bench.py --once --stats --layers 0,2 --passes fwd > gpurun_out/ncu_sel.log 2>&1
ncu -i /tmp/sel_full.ncu-rep --page raw --csv > gpurun_out/sel_raw.csv 2>/dev/null
ncu -i /tmp/sel_full.ncu-rep --page details --csv > gpurun_out/sel_details.csv 2>/dev/null
cp /tmp/sel_full.ncu-rep gpurun_out/ 2>/dev/null
cat gpurun_out/bench.json; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/conv_sel.txt
