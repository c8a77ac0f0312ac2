#!/bin/bash
# The round's evidence run on one B200: GPU tests, bench line, reference arm,
# per-config lines, the per-frame API numbers, the ncu launch list of the bench command,
# the red-op metrics and one full ncu capture of the top kernels.  Outputs in $1.
out=${1:-gpurun_out}
mkdir -p "$out"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > "$out/gputest.log" 2>&1; tail -3 "$out/gputest.log"
timeout 600 python bench.py --steps 10 --warmup 3 > "$out/bench.json" 2> "$out/bench.err"; tail -1 "$out/bench.json"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$out/bench_ref.json" 2> "$out/bench_ref.err"; tail -1 "$out/bench_ref.json"
timeout 900 python tools/bench_configs.py cfg1 cfg2 cfg2sum cfg4 cfg5 cfg2furn cfg2f64 cfg2fix > "$out/configs.jsonl" 2>&1
timeout 300 python tools/bench_session.py 2000 fixed64,float32,ann,lib > "$out/session.json" 2>&1
timeout 300 python tools/fallback_cost.py > "$out/fallback_cost.json" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches.csv" \
  python bench.py --frames 512 --steps 1 --warmup 1 --no-e2e --no-cpu --no-f64 > "$out/ncu_launch.log" 2>&1
bash tools/ncu_red.sh "$out" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_raster[^_]|k_raster$|k_ccsetup|k_fuse_fast" -s 4 -c 4 \
  -o "$out/full" python bench.py --frames 256 --steps 1 --warmup 1 --no-e2e --no-cpu --no-f64 > "$out/ncu_full.log" 2>&1
echo done
