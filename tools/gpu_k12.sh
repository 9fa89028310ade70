# k12 plan: parity tests at n = 16383/16385 + the benchmarked path, bench, per-stage cycles
timeout 900 python -m pytest tests/test_conv_gpu.py -x -q -k "16383 or 16385 or k12 or config2 or large_n or duplicate" > gpurun_out/k12_tests.log 2>&1; echo TESTS_RC $?; tail -3 gpurun_out/k12_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k12_bench.json 2> gpurun_out/k12_bench.err; echo BENCH_RC $?; tail -2 gpurun_out/k12_bench.err
python -c "import json;d=json.load(open('gpurun_out/k12_bench.json'));print('k12 ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'], d['validation']['parity']['max_rel_err'])"
TGB_PHASE_CLK=1 timeout 300 python tools/prof_pair.py > gpurun_out/k12_phase.log 2>&1; echo PHASE_RC $?; grep k12 gpurun_out/k12_phase.log | tail -1
