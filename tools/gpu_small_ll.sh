# launch lists of config 0 without cache flushes (ncu --cache-control none), per variant
for v in warp cta old; do
  unset TGB_NO_SMALL TGB_SMALL_CTA
  if [ $v = old ]; then export TGB_NO_SMALL=1; fi
  if [ $v = cta ]; then export TGB_SMALL_CTA=1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/cfg0_ll_$v.csv python tools/prof_cfg0.py > /dev/null 2>&1; echo NCU_RC $?
done
