for args in "--overlap 0" "--overlap 1 --fuse-ctas 1" "--overlap 1 --fuse-ctas 2" "--overlap 1 --fuse-ctas 3" "--overlap 1 --fuse-ctas 5" "--overlap 1 --fuse-ctas 0"; do
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$args', round(d['value']), round(d['roofline']['frac'],3), d['breakdown_ms_per_step'])"
done
