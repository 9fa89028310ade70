# A/B of an env knob on the rank reduction / TEI fit: usage bash tools/ab_red.sh "TGB_NO_SPLITK=1"
ALT="$1"
timeout 600 python -m pytest tests -x -q -m gpu -k "reduc or linalg or tei or hf or scf or golden" 2>&1 | tail -1
env $ALT timeout 600 python -m pytest tests -x -q -m gpu -k "reduc or linalg or tei or hf or scf or golden" 2>&1 | tail -1
for v in "" "$ALT" "" "$ALT"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py abr 1,3 2>&1 | grep '"config"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:round(d[k],2) for k in ('density_tensor_device_ms','reduce_rank_ms','fit_ms','cholesky_ms') if k in d})"
done
