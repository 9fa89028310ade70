for m in 0 1 2 4 3 5 6 7; do
  TGB_PAIR_DBG=$m python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('mode',$m,'pair_ms',round(d['roofline']['avg_launch_ms'],4))"
done
