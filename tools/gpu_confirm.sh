# final confirmation of the committed build: GPU tests, smoke, bench, reference arm
python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo TESTS_RC $?; tail -1 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo REF_RC $?
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo BENCH_RC $?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/final_bench.json").read().strip().splitlines()[-1])
print("bench", d["ms_per_step"], d["value"], d["roofline"]["frac"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "parity", d["validation"]["parity"]["max_rel_err"], d["clocks"])
r=json.loads(open("gpurun_out/final_ref.json").read().strip().splitlines()[-1])
print("ref", r["value"], r["ms_per_step"])
PY
