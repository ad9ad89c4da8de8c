# A/B of the tile-interleaved epilogue (NNL_EPI_IL) on the conv table and the bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_gemm_gpu.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_tc.log
tail -3 gpurun_out/pytest_tc.log
NNL_EPI_IL=0 timeout 300 python tools/conv_bench.py --stats > gpurun_out/conv_il0.txt 2>&1
timeout 300 python tools/conv_bench.py --stats > gpurun_out/conv_il1.txt 2>&1
NNL_EPI_IL=0 timeout 500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_il0.json 2> gpurun_out/bench_il0.err
timeout 500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_il1.json 2> gpurun_out/bench_il1.err
paste gpurun_out/conv_il0.txt gpurun_out/conv_il1.txt | awk -F'\t' '{printf "%-60s | %s\n", substr($1,1,60), substr($2,35,30)}'
cut -c1-330 gpurun_out/bench_il0.json gpurun_out/bench_il1.json
