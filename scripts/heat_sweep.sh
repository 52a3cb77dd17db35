# heat kernels (config 2: 2^28 f64, 1000 steps): OFL_HEAT_KERNEL 2 = warp
# tiles, one tile per warp; 4 = persistent warps with cp.async prefetch of
# the next tile.  OFL_HEAT_FMA=1 fused two-DFMA update (default) / 0 unfused;
# cells/thread R; temporal block tb.  Earlier kernels (0 CTA register tiles,
# 1 smem tiles, 3 two-level): profiles/r01_heat_sweep.txt.
for k in ${KERNELS:-4 2}; do
  for fma in ${FMAS:-1}; do
    for r in ${RS:-16 24 32}; do
      for tb in ${TBS:-48 64}; do
        echo "== OFL_HEAT_KERNEL=$k OFL_HEAT_FMA=$fma OFL_HEAT_R=$r tb=$tb"
        OFL_HEAT_KERNEL=$k OFL_HEAT_FMA=$fma OFL_HEAT_R=$r OFL_HEAT_TB=$tb python scripts/profile_kernels.py heat_time 2>&1 | tail -1
      done
    done
  done
done
