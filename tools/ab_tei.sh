# A/B of an env knob on the config-3 TEI Cholesky: usage bash tools/ab_tei.sh "TGB_TEI_SIMT_COLUMN=1"
ALT="$1"
timeout 600 python -m pytest tests -x -q -m gpu -k "tei or hf or scf" 2>&1 | tail -1
env $ALT timeout 600 python -m pytest tests -x -q -m gpu -k "tei or hf or scf" 2>&1 | tail -1
for v in "" "$ALT" "" "$ALT"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py abt 3 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print({k:d[k] for k in ('fit_ms','conv_ms','cholesky_ms','R_B')})"
done
