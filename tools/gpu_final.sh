# full default bench (device value, e2e, cpu baseline, clocks) + reference arm + launch list
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo BENCH_RC $?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo REF_RC $?
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1
echo NCU_RC $?
