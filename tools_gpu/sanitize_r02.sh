# GPU box: compute-sanitizer racecheck / synccheck / memcheck over one small projector that runs the
# mbarrier, named-barrier and warp-specialised kernels (k_leaf_chol4, k_core_any, k_tsqr, k_apply,
# k_hsolve2), direct launches (no graph) so reports name the kernel
mkdir -p gpurun_out
cat > /tmp/san_one.py <<'P'
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1608_01164_b200 as S
A = S.dimer_chain(int(sys.argv[1]), 1.0, 0.9, 0.1, 3)
r = S.hqdwh(A, int(sys.argv[2]), 1e-10)
print("iterations", r.iterations, "trace", r.info["trace"], "max_rank", r.info["max_rank"], flush=True)
r.close()
B = S.dimer_chain(1536, 1.0, 0.8, 0.0, 5, b=4, s=0.01)
r = S.hqdwh(B, 128, 1e-10)
print("banded iterations", r.iterations, "trace", r.info["trace"], flush=True)
r.close()
P
for tool in racecheck synccheck memcheck; do
  SPG_NO_GRAPH=1 SPG_NO_PLAN_CACHE=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 \
     python /tmp/san_one.py 2048 256 > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|iterations" gpurun_out/sanitizer_$tool.log | tail -4
done
