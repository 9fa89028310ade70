# config-0 latency A/B over the generic kernels' CTA widths
for pt in 0 32 96; do
  TGB_PAIR_THREADS=$pt timeout 120 python tools/bench_configs.py ab 0 > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_configs.json'))[0];print('pair',$pt,'host_ms',round(d['ms'],4),'dev_ms',round(d['device_ms_per_call'],4))"
done
