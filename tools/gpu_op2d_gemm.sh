# 2D operator as element GEMM (STGMG_OP2D_GEMM=1) vs the register sum-factorised op2d: per-level K1 / sweep times
echo "op2d: $(timeout 300 python tools/kernel_times.py --config ${CFG:-1} 2>&1 | grep -E 'level (5|4) |vcycle' | sed 's/K2.*sweep/sweep/' | tr '\n' ' ')"
for v in ${VARS:-0 1 2 7}; do
  echo "gemm v=$v: $(STGMG_OP2D_GEMM=1 STGMG_EK2_VARIANT=$v timeout 300 python tools/kernel_times.py --config ${CFG:-1} 2>&1 | grep -E 'level (5|4) |vcycle' | sed 's/K2.*sweep/sweep/' | tr '\n' ' ')"
done
