timeout 600 python -m pytest tests/test_tei_gpu.py tests/test_hf_gpu.py -x -q 2>&1 | tail -2
timeout 300 python tools/bench_configs.py s2c 3 2>&1 | tail -1
cat > /tmp/tei_prof.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case
bs,_=basis_case(3); disc=tg.discretize_basis(bs)
kern=tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[3], KERNEL_C0[3]), False)
ctx=tg.Context(0)
f=tg.TEIFactorization(ctx); tg.tei_density_fitting(f,bs,disc,1e-6); tg.tei_convolution_matrices(f,kern); tg.tei_cholesky(f,1e-6)
torch.cuda.synchronize(); print("ok", f.rank_b())
PY
TGB_TEI_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv python /tmp/tei_prof.py 2>/dev/null | python tools/ncu_sum.py
