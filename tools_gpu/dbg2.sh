mkdir -p gpurun_out
T="tests/test_gpu_parity.py -x -q -k not_first_iterate_and_not_stacked"
for v in "SPG_X=1" "SPG_DBG_LR_OLD=1" "SPG_DBG_NO_EARLY=1" "SPG_FIRST_ITERATE=cholesky" "SPG_NO_PLAN_CACHE=1"; do
  echo "== $v"; env $v python -m pytest tests/test_gpu_parity.py -x -q -k "not first_iterate and not stacked and not baseline" 2>&1 | tail -2
done
cat > /tmp/ic.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import make_input
c = dict(n=4096, b=1, t1=1.0, t2=0.999, eps_dis=2e-4, s=0.0, nmin=256, eps=1e-10, seed=2)
r = S.hqdwh(make_input(c), 256, 1e-10); print(r.iterations, r.info["trace"])
PY
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python /tmp/ic.py > gpurun_out/initcheck.log 2>&1; tail -60 gpurun_out/initcheck.log
