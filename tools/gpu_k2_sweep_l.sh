# K2 tile-variant sweep on the middle levels of cfg1 (kernel_times.py lines of levels 4 and 3)
for v in 0 1 2 6 4 7 8; do for dn in 0 1; do
  echo "v=$v dense=$dn:"; STGMG_K2_VARIANT_L4=$v STGMG_K2_VARIANT_L3=$v STGMG_K2_DENSE=$dn timeout 300 python tools/kernel_times.py --config ${CFG:-1} 2>&1 | grep -E 'level (4|3)|vcycle'
done; done
