for env in "" "RK_BP_NARROW=0" "RK_BP_WIDE_GROUPS=0" "RK_SINGLE_LANE=0" "RK_BP_NARROW=0 RK_BP_WIDE_GROUPS=0"; do
  echo "== env: $env"
  env $env RK_STRESS_ONLY=179,285,322,465 timeout 300 python tools/stress_parity.py 600 2 520 2>&1 | tail -9
done
