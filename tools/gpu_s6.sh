# session-6 evidence: full GPU tests, bench, reference arm, smoke, launch list, ncu --set full of the pair kernel, scale probe, configs
python -m pytest tests -m gpu -x -q > gpurun_out/s6_tests.log 2>&1; echo TESTS_RC $?; tail -2 gpurun_out/s6_tests.log
python bench.py > gpurun_out/s6_bench.json 2> gpurun_out/s6_bench.err; echo BENCH_RC $?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s6_ref.json 2> gpurun_out/s6_ref.err; echo REF_RC $?
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s6_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s6_ncu.log 2>&1
echo NCU_RC $?
python tools/prof_pair.py 500 > gpurun_out/s6_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k12_pair_kernel -s 1 -c 1 -o gpurun_out/s6_k12 -f python tools/prof_pair.py 500 > gpurun_out/s6_k12.log 2>&1
echo NCUFULL_RC $?
TGB_PHASE_CLK=1 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "k12 " | tail -2 > gpurun_out/s6_phase.txt; cat gpurun_out/s6_phase.txt
python tools/scale_probe.py > gpurun_out/s6_scale_probe.txt 2>&1; tail -8 gpurun_out/s6_scale_probe.txt
python tools/bench_configs.py > gpurun_out/s6_configs.json 2> gpurun_out/s6_configs.err; echo CONFIGS_RC $?
