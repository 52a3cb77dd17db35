# heat kernels: OFL_HEAT_KERNEL (0 CTA-register, 2 warp-independent, 3 two-level) x cells/thread
for cfg in "OFL_HEAT_KERNEL=3" "OFL_HEAT_KERNEL=2 OFL_HEAT_R=24" "OFL_HEAT_KERNEL=2 OFL_HEAT_R=16"; do
  for tb in 40 48 56 64; do
    echo "== $cfg tb=$tb"; env $cfg OFL_HEAT_TB=$tb python scripts/profile_kernels.py heat_time 2>&1 | tail -1
  done
done
