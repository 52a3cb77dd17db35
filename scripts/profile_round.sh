set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/bench_configs.py --out gpurun_out/configs.json > /dev/null 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
N="ncu --set full --clock-control none --import-source on"
$N -k regex:k_mandelbrotP -s 1 -c 1 -o gpurun_out/r01b_mandel python scripts/profile_kernels.py mandel > gpurun_out/ncu_mandel.log 2>&1
$N -k regex:k_heat_warp -s 1 -c 1 -o gpurun_out/r01b_heat python scripts/profile_kernels.py heat > gpurun_out/ncu_heat.log 2>&1
$N -k regex:k_sum -s 1 -c 1 -o gpurun_out/r01b_sum python scripts/profile_kernels.py sum > gpurun_out/ncu_sum.log 2>&1
ls gpurun_out
