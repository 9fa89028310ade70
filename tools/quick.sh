# quick perf+parity cycle: conv/golden tests, phase clocks, bench, launch list
timeout 600 python -m pytest tests -x -q -m gpu -k "conv or golden or smoke" 2>&1 | tail -1
TGB_PHASE_CLK=1 timeout 120 python tools/prof_pair.py 2>&1 | grep "phase cycles" | tail -2 | head -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python -c "import json,sys;d=json.load(open('gpurun_out/quick_bench.json'));print('ms',round(d['ms_per_step'],4),'pair_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],4))" || tail -5 gpurun_out/quick_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spectrum|pair|dup|build" -c 15 --csv python tools/prof_pair.py 2>/dev/null | python tools/ncu_sum.py
