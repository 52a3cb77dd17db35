set -x
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
$N -k regex:k_stream_tile -s 1 -c 1 -o gpurun_out/r01_triad python scripts/profile_kernels.py triad > gpurun_out/ncu_triad.log 2>&1
$N -k regex:k_mandelbrot -s 1 -c 1 -o gpurun_out/r01_mandel python scripts/profile_kernels.py mandel > gpurun_out/ncu_mandel.log 2>&1
$N -k regex:k_heat_reg -s 1 -c 1 -o gpurun_out/r01_heat python scripts/profile_kernels.py heat > gpurun_out/ncu_heat.log 2>&1
$N -k regex:k_stencil -s 1 -c 1 -o gpurun_out/r01_stencil python scripts/profile_kernels.py stencil > gpurun_out/ncu_stencil.log 2>&1
$N -k regex:k_dot -s 1 -c 1 -o gpurun_out/r01_dot python scripts/profile_kernels.py dot > gpurun_out/ncu_dot.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 200 --warmup 5 --no-overhead --cpu-seconds 0 --e2e-steps 2 > /dev/null 2>&1
ls -la gpurun_out | tail -12
