# split-raster A/B on one box (DESIGN "tried"): bash tools/split_ab.sh
for rep in 1 2; do
for args in "--split-raster 0" "--split-raster 1" "--split-raster 1 PRIO=-1"; do
  prio=0; case "$args" in *PRIO=-1*) prio=-1;; esac
  a=${args% PRIO=-1}
  TFB_SPLIT_PRIO=$prio python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-f64 --no-render $a 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$args', round(d['value']), round(d['roofline']['frac'],3), {k: round(v,2) for k,v in d['breakdown_ms_per_step'].items()})"
done
done
