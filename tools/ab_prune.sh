#!/bin/bash
# A/B of the band-limited pruning in k12_pair_kernel (run under gpurun)
set -x
mkdir -p gpurun_out
python -m pytest tests/test_conv_gpu.py tests/test_coverage_gpu.py tests/test_spectrum_gpu.py -m gpu -x -q > gpurun_out/prune_tests.log 2>&1
tail -5 gpurun_out/prune_tests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/prune_bench.json 2> gpurun_out/prune_bench.err
TGB_K12_NO_PRUNE=1 python bench.py --steps 20 --warmup 3 > gpurun_out/noprune_bench.json 2> gpurun_out/noprune_bench.err
TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 2>&1 | grep "k12 cycles" | tail -2 > gpurun_out/prune_phase.txt
TGB_K12_NO_PRUNE=1 TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 2>&1 | grep "k12 cycles" | tail -2 > gpurun_out/noprune_phase.txt
python - <<'PY'
import json
for f in ("prune","noprune"):
    try:
        d=json.loads(open(f"gpurun_out/{f}_bench.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"], d.get("parity"), d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e, open(f"gpurun_out/{f}_bench.err").read()[-2000:])
PY
cat gpurun_out/prune_phase.txt gpurun_out/noprune_phase.txt
