# K2L experiments on cfg1 level 4 / 3: tile variant x tile-count target (kernel_times.py level lines)
for v in 7 4 8; do for tt in 0 888 1184 1776; do
  if [ $tt = 0 ]; then unset STGMG_TILE_TARGET; else export STGMG_TILE_TARGET=$tt; fi
  echo "v=$v tt=$tt: $(STGMG_K2_VARIANT_L4=$v STGMG_K2_VARIANT_L3=$v timeout 300 python tools/kernel_times.py 2>&1 | grep -E 'level (4|3)' | cut -c1-60 | tr '\n' ' ')"
done; done
