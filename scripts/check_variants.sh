# Parity of every sweep variant kept in the kernels (the defaults run in the
# normal GPU suite).  Run on the GPU box: bash scripts/check_variants.sh
P="timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider"
for k in 0 1 3; do echo "OFL_HEAT_KERNEL=$k: $(OFL_HEAT_KERNEL=$k $P -k heat 2>&1 | tail -1)"; done
echo "OFL_HEAT_FMA=0: $(OFL_HEAT_FMA=0 $P -k heat 2>&1 | tail -1)"
for v in 1 2 3 4 5 6; do echo "OFL_STENCIL2D_VARIANT=$v: $(OFL_STENCIL2D_VARIANT=$v $P -k 'stencil2d or heat2d' 2>&1 | tail -1)"; done
for v in 1 2 3 4 5 7; do echo "OFL_STENCIL_VARIANT=$v: $(OFL_STENCIL_VARIANT=$v $P -k 'stencil and not 2d' 2>&1 | tail -1)"; done
for v in 0 19 5 10 11 12 16 17; do echo "OFL_STREAM_VARIANT=$v: $(OFL_STREAM_VARIANT=$v $P -k 'stream or triad' 2>&1 | tail -1)"; done
for e in "OFL_MANDEL_PERIOD=0" "OFL_MANDEL_FUSED=0" "OFL_MANDEL_ILP=2" "OFL_MANDEL_ILP=1" "OFL_MANDEL_FPCMP=1"; do
  echo "$e: $(env $e $P -k mandel 2>&1 | tail -1)"; done
for c in 1 2 4; do echo "OFL_REDUCE_CPS=$c: $(OFL_REDUCE_CPS=$c $P -k 'sum or dot' 2>&1 | tail -1)"; done
