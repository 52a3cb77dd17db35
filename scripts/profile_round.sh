# One GPU call: GPU tests, BASELINE configs, ncu --set full of the top kernels,
# compute-sanitizer.  Outputs land in gpurun_out/ (copy summaries to profiles/);
# P (default rp) prefixes the capture names.
set -x
mkdir -p gpurun_out
P=${P:-rp}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/bench_configs.py --out gpurun_out/configs.json > /dev/null 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
N="ncu --set full --clock-control none --import-source on"
$N -k regex:k_stream_tile -s 1 -c 1 -o gpurun_out/${P}_triad python scripts/profile_kernels.py triad > gpurun_out/ncu_triad.log 2>&1
$N -k regex:k_mandelbrotP -s 1 -c 1 -o gpurun_out/${P}_mandel python scripts/profile_kernels.py mandel > gpurun_out/ncu_mandel.log 2>&1
OFL_MANDEL_PERIOD=0 $N -k regex:k_mandelbrotP -s 1 -c 1 -o gpurun_out/${P}_mandel_plain python scripts/profile_kernels.py mandel > gpurun_out/ncu_mandel_plain.log 2>&1
$N -k regex:k_stencil2d -s 2 -c 1 -o gpurun_out/${P}_stencil2d python scripts/bench_configs.py --only stencil2d > /dev/null 2>&1
# the third pass of config 2 (a production pass of ~83 steps, not the first)
$N -k regex:k_heat_pipe -s 2 -c 1 -o gpurun_out/${P}_heat python scripts/profile_kernels.py heat 1 > gpurun_out/ncu_heat.log 2>&1
$N -k regex:k_dot -s 1 -c 1 -o gpurun_out/${P}_dot python scripts/profile_kernels.py dot > gpurun_out/ncu_dot.log 2>&1
$N -k regex:k_sum -s 1 -c 1 -o gpurun_out/${P}_sum python scripts/profile_kernels.py sum > gpurun_out/ncu_sum.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${P}_bench_launches.csv python bench.py --steps 200 --warmup 5 --configs "" --no-overhead --cpu-seconds 0 --e2e-steps 2 > /dev/null 2>&1
bash scripts/sanitize.sh > gpurun_out/sanitizer.txt 2>&1
ls gpurun_out
