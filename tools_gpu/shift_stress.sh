for env in "" "SPG_NO_PLAN_CACHE=1" "SPG_DBG_POISON=1" "SPG_DBG_POISON=1 SPG_NO_PLAN_CACHE=1"; do
  echo "== env: $env"
  env $env python tools_gpu/shift_stress.py 40 2>&1 | grep -E "failures"
done
