# A/B of one environment switch of libtgb on the bench: usage bash tools/ab_env.sh VAR=VALUE [reps]
for i in $(seq 1 ${2:-2}); do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab0.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab0.json'));print('base   ', round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4), d['validation']['parity']['max_rel_err'])"
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab1.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab1.json'));print('$1', round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4), d['validation']['parity']['max_rel_err'])"
done
env $1 TGB_PHASE_CLK=1 timeout 300 python tools/prof_pair.py 2>&1 | grep k12 | tail -1
