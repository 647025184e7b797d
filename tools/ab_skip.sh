for v in "" lane grp merge fin classify "lane,grp" "lane,grp,merge"; do
  A3G_DIAG_SKIP=$v A3G_DIAG_SKIP_COMPUTE=1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip [$v] sampling-only', round(d['ms_per_step'],4))"
done
