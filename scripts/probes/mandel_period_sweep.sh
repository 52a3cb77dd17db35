# Probe: the cycle-test interval (OFL_PERIOD_CHECK) of the production Mandelbrot kernel, rebuilt on
# the GPU box per value; prints the config-3 kernel time and the parity tests.
cp paper_1810_11482_b200/csrc/k_mandelbrot.cu /tmp/km_orig.cu
for K in 8 16 32; do
  sed -e "s/#define OFL_PERIOD_CHECK 16/#define OFL_PERIOD_CHECK $K/" /tmp/km_orig.cu > paper_1810_11482_b200/csrc/k_mandelbrot.cu
  make -s -C paper_1810_11482_b200/csrc -j 16 > /tmp/mk.log 2>&1 || { echo "build failed: $K"; continue; }
  echo "check every $K: $(python scripts/probes/mandel_setup_cost.py | grep '^2000') / $(python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k 'mandelbrot' 2>&1 | tail -1)"
done
cp /tmp/km_orig.cu paper_1810_11482_b200/csrc/k_mandelbrot.cu
make -s -C paper_1810_11482_b200/csrc -j 16 > /dev/null 2>&1
