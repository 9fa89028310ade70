# test + bench + launch list in one gpurun call.  usage: bash tools/gpu_cycle.sh TAG [pytest-args]
TAG=${1:-cyc}; shift
timeout 900 python -m pytest tests -x -q -m gpu "$@" > gpurun_out/${TAG}_tests.log 2>&1; echo TESTS_RC $? ; tail -3 gpurun_out/${TAG}_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo BENCH_RC $?
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print('ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'])"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo NCU_RC $?
