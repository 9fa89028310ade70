# round-2 checkpoint: full GPU suite, smoke, bench (with e2e + CPU baseline), launch list
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/full_tests.log 2>&1; echo TESTS_RC $?; tail -3 gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo BENCH_RC $?; tail -2 gpurun_out/full_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/full_ref.json 2> gpurun_out/full_ref.err; echo REF_RC $?
