# Probe: Mandelbrot queue unit (tiles per pop) and warp tile shape at the production P, rebuilt
# on the GPU box per variant; prints the config-3 kernel time and the parity tests.

cp paper_1810_11482_b200/csrc/k_mandelbrot.cu /tmp/km_orig.cu
for cfg in "4 8 4" "2 8 4" "8 8 4" "4 4 8" "4 16 2"; do
  set -- $cfg
  U=$1; TW=$2; TH=$3
  sed -e "s/constexpr int kTilesPerUnit = 4;/constexpr int kTilesPerUnit = $U;/" \
      -e "s/constexpr int kTileW = 8, kTileH = 4;/constexpr int kTileW = $TW, kTileH = $TH;/" /tmp/km_orig.cu > paper_1810_11482_b200/csrc/k_mandelbrot.cu
  make -s -C paper_1810_11482_b200/csrc -j 16 > /tmp/mk.log 2>&1 || { echo "build failed: $cfg"; tail -3 /tmp/mk.log; continue; }
  echo "unit=$U tile=${TW}x$TH: $(python scripts/probes/mandel_setup_cost.py | grep '^2000') / $(python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k 'mandelbrot' 2>&1 | tail -1)"
done
cp /tmp/km_orig.cu paper_1810_11482_b200/csrc/k_mandelbrot.cu
