# compute-sanitizer racecheck / synccheck / memcheck over the tcgen05 paths:
# halo tiles (fwd/dgrad), halo weight gradients (64- and 128-wide blocks), 256-wide
# and CTA-pair tiles, strided-dgrad parity classes, the stem (space-to-depth, x4 halo
# wgrad), split-K reductions.  Writes gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
SEL="geom1 or geom5 or geom13 or geom15 or geom17 or geom19"
for tool in racecheck synccheck memcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
    python -m pytest tests/test_tc_gemm_gpu.py -q -p no:cacheprovider -k "$SEL" \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
  tail -3 gpurun_out/sanitize_$tool.txt
done
