for v in "OFL_MANDEL_ILP=2" "OFL_MANDEL_ILP=4" "OFL_MANDEL_ILP=8"; do
  echo "== $v"; env $v python scripts/bench_configs.py --only mandel 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin)['config3_mandelbrot']; print(d['kernel_ms'], d['frac_fp64'], d['sha256_matches_reference'], d['fp64_peak_measured_tops'])"
done
