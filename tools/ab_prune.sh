#!/bin/bash
# A/B of a k12_pair_kernel switch (run under gpurun): tools/ab_prune.sh TGB_K12_NO_DEFER [notests]
V=${1:-TGB_K12_NO_PRUNE}
mkdir -p gpurun_out
if [ "$2" != "notests" ]; then
python -m pytest tests/test_conv_gpu.py tests/test_coverage_gpu.py tests/test_spectrum_gpu.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -5 gpurun_out/ab_tests.log
fi
python bench.py --steps 20 --warmup 3 > gpurun_out/ab_on.json 2> gpurun_out/ab_on.err
env $V=1 python bench.py --steps 20 --warmup 3 > gpurun_out/ab_off.json 2> gpurun_out/ab_off.err
TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 2>&1 | grep "k12 cycles" | tail -1 > gpurun_out/ab_on_phase.txt
env $V=1 TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 2>&1 | grep "k12 cycles" | tail -1 > gpurun_out/ab_off_phase.txt
python - <<'PY'
import json
for f in ("on","off"):
    try:
        d=json.loads(open(f"gpurun_out/ab_{f}.json").read().strip().splitlines()[-1])
        print(f, "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "launch ms", d["roofline"]["avg_launch_ms"], "parity", d.get("validation",{}).get("parity"), "e2e", d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e, open(f"gpurun_out/ab_{f}.err").read()[-2000:])
PY
cat gpurun_out/ab_on_phase.txt gpurun_out/ab_off_phase.txt
