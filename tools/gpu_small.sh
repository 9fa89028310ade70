# small-plan kernels (config 0 / config 1 sizes): parity, config-0 A/B, launch list
timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_hf_gpu.py tests/test_golden.py tests/test_tei_gpu.py -x -q -m gpu > gpurun_out/small_tests.log 2>&1; echo TESTS_RC $?; tail -3 gpurun_out/small_tests.log
for v in new old new old; do
  unset TGB_NO_SMALL
  if [ $v = old ]; then export TGB_NO_SMALL=1; fi
  timeout 300 python tools/bench_configs.py ab 0,1 > /dev/null 2> gpurun_out/small_ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_configs.json'));print('$v',[(x.get('config'),x.get('device_ms_per_call'),x.get('launches_per_call'),x.get('parity_factor_relmax'),x.get('hartree_ms')) for x in d])"
done
unset TGB_NO_SMALL
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/cfg0_ll_new.csv python tools/prof_cfg0.py > /dev/null 2>&1; echo NCU_RC $?
