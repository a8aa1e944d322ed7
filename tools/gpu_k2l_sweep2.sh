# K2L variant sweep on cfg1 levels 1-3 (kernel_times.py level lines)
for v in 4 7 8; do
  echo "v=$v: $(STGMG_K2_VARIANT_L1=$v STGMG_K2_VARIANT_L2=$v STGMG_K2_VARIANT_L3=$v timeout 300 python tools/kernel_times.py 2>&1 | grep -E 'level (3|2|1) ' | cut -c1-44 | tr '\n' ' ')"
done
