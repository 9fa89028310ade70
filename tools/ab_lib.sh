# A/B of two in-tree builds: usage bash tools/ab_lib.sh libtgb_u2.so
ALT=${1:-libtgb_u2.so}
TGB_LIB=$ALT timeout 600 python -m pytest tests -x -q -m gpu -k "conv or golden" 2>&1 | tail -1
for L in libtgb.so $ALT libtgb.so $ALT; do
  echo "== $L"
  TGB_LIB=$L TGB_PHASE_CLK=1 timeout 120 python tools/prof_pair.py 2>&1 | grep "phase cycles" | tail -2 | head -1
  TGB_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json,sys;d=json.load(open('gpurun_out/x.json'));print('ms',round(d['ms_per_step'],4),'pair_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],4))" || tail -5 gpurun_out/x.err
done
