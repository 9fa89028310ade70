# full GPU suite (+ the 2-process sharding test three times), bench
for i in 1 2 3; do timeout 600 python -m pytest tests/test_sharding_gpu.py -x -q > gpurun_out/r2c_shard_$i.log 2>&1; echo SHARD_RC $?; done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2c_tests.log 2>&1; echo TESTS_RC $?; tail -5 gpurun_out/r2c_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo BENCH_RC $?; tail -2 gpurun_out/r2c_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2c_bench.json'));print('ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'], d['validation']['parity']['max_rel_err'], 'e2e', d['e2e']['value'])"
