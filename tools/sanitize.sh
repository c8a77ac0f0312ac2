#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the smoke workload (every
# hot-path kernel: cluster cull, setup, tile raster, scatter-add fast + general,
# finalize, render) and two small GPU test files.  Logs under $1 (default gpurun_out/).
out=${1:-gpurun_out}
mkdir -p "$out"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python -c "import __graft_entry__ as g; g.smoke()" > "$out/sanitize_${tool}_smoke.log" 2>&1
  echo "$tool smoke rc=$?" >> "$out/sanitize_summary.txt"
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 \
  python -m pytest -q -p no:cacheprovider tests/test_gpu_fixed.py tests/test_gpu_finalize.py \
  > "$out/sanitize_memcheck_tests.log" 2>&1
echo "memcheck tests rc=$?" >> "$out/sanitize_summary.txt"
cat "$out/sanitize_summary.txt"
