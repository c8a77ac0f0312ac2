# compare the current tree with the tree in _exp/old (both with their own library)
for rep in 1 2; do
for t in . _exp/old; do
  (cd $t && python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); b=d['breakdown_ms_per_step']; n=d['config']['frames_per_gpu']; print('$t', round(d['value']), {k: round(v/n*1000,3) for k,v in b.items()})")
done
done
for t in . _exp/old; do (cd $t && python tools/bench_configs.py cfg5 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$t cfg5', round(d['frames_per_s']), round(d['raster_us_per_frame'],2), round(d['fuse_us_per_frame'],2))"); done
