for b in 256 64 32 16; do
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --batch $b 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); b=d['breakdown_ms_per_step']; n=d['config']['frames_per_gpu']; print('$b', round(d['value']), {k: round(v/n*1000,3) for k,v in b.items()})"
done
