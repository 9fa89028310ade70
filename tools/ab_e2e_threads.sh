for t in 16 8 4 12 16; do
  TGB_COPY_THREADS=$t timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('threads $t e2e ms', round(d['e2e']['ms_per_step'],1))"
done
