# k12 plan: parity tests at n = 16383/16385, then bench new vs old path, then the launch list
timeout 900 python -m pytest tests/test_conv_gpu.py -x -q -k "16383 or 16385 or k12 or config2 or large_n" > gpurun_out/k12_tests.log 2>&1; echo TESTS_RC $?; tail -15 gpurun_out/k12_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k12_bench.json 2> gpurun_out/k12_bench.err; echo BENCH_RC $?; tail -3 gpurun_out/k12_bench.err
python -c "import json;d=json.load(open('gpurun_out/k12_bench.json'));print('k12 ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'], d['validation']['parity'])"
TGB_NO_K12=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k12_bench_old.json 2> gpurun_out/k12_bench_old.err; echo BENCH_OLD_RC $?
python -c "import json;d=json.load(open('gpurun_out/k12_bench_old.json'));print('old ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'])"
#timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/k12_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k12_ncu.log 2>&1; echo NCU_RC $?
