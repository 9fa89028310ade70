# quick check of a k12 kernel change (run under gpurun): the k12 tests, three bench lines, stage cycles
timeout 600 python -m pytest tests/test_conv_gpu.py -m gpu -x -q -k "k12 or config2" 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['validation']['parity']['max_rel_err'])"; done
TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "k12 " | tail -2
