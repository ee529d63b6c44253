# compute-sanitizer over the kernels added this round (small shapes)
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python tools/gpu/sanitize.py 2>&1 | tail -8
for tool in memcheck racecheck synccheck; do
  TILEFFT_NO_GRAPH=1 timeout 1500 $CS --tool $tool --print-limit 20 python tools/gpu/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
