# A/B of library variants on one box: bash tools/ab.sh default _exp/NAME.so ...
set -e
python -m pytest tests -m gpu -x -q -k "raster or parity or golden or smoke" 2>&1 | tail -1
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then unset TFB_LIB; else export TFB_LIB=$v; fi
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); b=d['breakdown_ms_per_step']; n=d['config']['frames_per_gpu']; print('$v', round(d['value']), {k: round(v/n*1000,3) for k,v in b.items()})"
done
done
