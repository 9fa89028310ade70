# A/B of the k12 pair kernels: parity at the benchmarked shape, bench, per-phase cycles.
# usage: bash tools/gpu_var.sh "bulk nobulk m1"   (bulk = default; nobulk = TGB_K12_NO_BULK=1; vN = TGB_K12_VAR=N; mN = TGB_K12_MODE=N)
mkdir -p gpurun_out
for V in ${1:-bulk nobulk}; do
  unset TGB_K12_VAR TGB_K12_NO_SHIFT TGB_K12_MODE TGB_K12_BULK
  case $V in noshift) export TGB_K12_NO_SHIFT=1;; bulk*) export TGB_K12_BULK=1;; v*) export TGB_K12_VAR=${V#v};; m*) export TGB_K12_MODE=${V#m};; esac
  if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_conv_gpu.py -x -q -k "16383 or 16385 or k12 or config2 or deterministic or duplicate or twin" > gpurun_out/var_${V}_tests.log 2>&1; echo VAR $V TESTS_RC $?; tail -2 gpurun_out/var_${V}_tests.log
  fi
  for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_${V}_bench.json 2> gpurun_out/var_${V}_bench.err; echo BENCH_RC $?
  python -c "import json;d=json.load(open('gpurun_out/var_${V}_bench.json'));print('VAR $V ms/step',d['ms_per_step'],'frac',d['roofline']['frac'],'pair_ms',d['roofline']['avg_launch_ms'], d['validation']['parity']['max_rel_err'])"
  done
  TGB_PHASE_CLK=1 timeout 300 python tools/prof_pair.py 2>&1 | grep k12 | tail -1
done
