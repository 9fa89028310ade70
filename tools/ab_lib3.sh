# A/B of pair-kernel time only (bench parity gate off: experimental builds may write wrong outputs)
for i in 1 2; do for L in libtgb.so $1; do
  TGB_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$L', round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4))" 2>/dev/null || echo "$L failed"
done; done
TGB_LIB=$1 TGB_PHASE_CLK=1 timeout 300 python tools/prof_pair.py 2>&1 | grep k12 | tail -1
