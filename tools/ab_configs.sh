# A/B of library variants on bench_configs: bash tools/ab_configs.sh CFG default _exp/NAME.so ...
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then unset TFB_LIB; else export TFB_LIB=$v; fi
  python tools/bench_configs.py $cfg | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['config'], round(d['frames_per_s']), 'raster', round(d['raster_us_per_frame'],2), 'fuse', round(d['fuse_us_per_frame'],2))"
done
