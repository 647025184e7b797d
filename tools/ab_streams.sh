for rep in 1 2; do for p in 8 12 16; do
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline --pipeline $p 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep', 'c2 streams $p', round(d['ms_per_step'],4), '%.3g'%d['value'])"
  python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline --pipeline $p 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep', 'c3 streams $p', round(d['ms_per_step'],4), '%.3g'%d['value'])"
done; done
