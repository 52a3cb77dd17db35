# Mandelbrot (config 3) variants: pixels per thread in lock step (OFL_MANDEL_ILP 1/2/3/4),
# exact cycle detection on/off (OFL_MANDEL_PERIOD), fused zi update on/off (OFL_MANDEL_FUSED).
for v in "OFL_MANDEL_ILP=4" "OFL_MANDEL_ILP=2" "OFL_MANDEL_PERIOD=0" "OFL_MANDEL_PERIOD=0 OFL_MANDEL_FUSED=0"; do
  echo "== $v"; env $v python scripts/probes/mandel_clock.py
done
