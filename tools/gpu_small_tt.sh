# config-0 pair kernel: CTA width A/B (TGB_SMALL_TT), device time per hartree_potential call
for rep in 1 2; do
for tt in 160 128 96 64; do
  TGB_SMALL_TT=$tt timeout 300 python tools/bench_configs.py ab 0 > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_configs.json'))[0];print('tt $tt', round(d['device_ms_per_call']*1e3,1), 'us', d['parity_factor_relmax'])"
done; done
