# A/B of an env knob on the config-2 pair kernel: usage bash tools/ab_env.sh "TGB_NO_FUSED=1"
ALT="$1"
timeout 600 python -m pytest tests -x -q -m gpu -k "conv or golden" 2>&1 | tail -1
env $ALT timeout 600 python -m pytest tests -x -q -m gpu -k "conv or golden" 2>&1 | tail -1
for v in "" "$ALT" "" "$ALT"; do
  echo "== $v"
  env $v TGB_PHASE_CLK=1 timeout 120 python tools/prof_pair.py 2>&1 | grep "phase cycles" | tail -2 | head -1
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json,sys;d=json.load(open('gpurun_out/x.json'));print('ms',round(d['ms_per_step'],4),'pair_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],4))" || tail -5 gpurun_out/x.err
done
