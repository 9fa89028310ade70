# alternating A/B of two in-tree builds on one box: bash tools/ab_lib4.sh libtgb_x.so
ALT=${1:-libtgb_u2.so}
for L in libtgb.so $ALT libtgb.so $ALT libtgb.so $ALT; do
  TGB_LIB=$L timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/x.json').read().strip().splitlines()[-1]);print('$L','ms',round(d['ms_per_step'],4),'pair_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],4))" || tail -5 gpurun_out/x.err
done
