# Probe: Mandelbrot pixels per thread (P) x min CTAs/SM of the PERIOD tile kernel, rebuilt on the
# GPU box per variant; prints the config-3 kernel time and the parity tests. Restores the source.
set -e
cp paper_1810_11482_b200/csrc/k_mandelbrot.cu /tmp/km_orig.cu
for cfg in "4 3" "2 3" "2 4" "2 6" "1 4" "1 8" "3 3"; do
  set -- $cfg
  P=$1; MB=$2
  sed -e "s/PERIOD ? 3 : 1) k_mandelbrotP/PERIOD ? $MB : 1) k_mandelbrotP/" \
      -e "s/k_mandelbrotP<true, 4, true>/k_mandelbrotP<true, $P, true>/" \
      -e "s/k_mandelbrotP<false, 4, true>/k_mandelbrotP<false, $P, true>/" /tmp/km_orig.cu > paper_1810_11482_b200/csrc/k_mandelbrot.cu
  if [ "$P" = "3" ]; then sed -i "s/constexpr int kTilesPerUnit = 4;/constexpr int kTilesPerUnit = 3;/" paper_1810_11482_b200/csrc/k_mandelbrot.cu; fi
  make -s -C paper_1810_11482_b200/csrc -j 16 > /dev/null 2>&1
  echo "P=$P minblocks=$MB: $(python scripts/probes/mandel_setup_cost.py | grep '^2000') / $(python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k 'mandelbrot_full or cycle_detection' 2>&1 | tail -1)"
done
cp /tmp/km_orig.cu paper_1810_11482_b200/csrc/k_mandelbrot.cu
