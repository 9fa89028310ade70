# round-2 first GPU pass: full GPU suite (incl. the config-2 full-path parity test) + bench
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_tests.log 2>&1; echo TESTS_RC $?; tail -5 gpurun_out/r2a_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo BENCH_RC $?
tail -3 gpurun_out/r2a_bench.err
nproc
