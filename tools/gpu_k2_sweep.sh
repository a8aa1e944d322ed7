# cfg1 fine-level K2 variant / dense / tile-target sweep (kernel_times.py, fine level line only)
for v in 1 2 6; do for dn in 0 1; do for tt in 0 296 444 592; do
  if [ $tt = 0 ]; then unset STGMG_TILE_TARGET; else export STGMG_TILE_TARGET=$tt; fi
  echo "v=$v dense=$dn tt=$tt: $(STGMG_K2_VARIANT=$v STGMG_K2_DENSE=$dn timeout 300 python tools/kernel_times.py --config ${CFG:-1} 2>&1 | grep -m1 'level' )"
done; done; done
