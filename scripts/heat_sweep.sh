# heat kernels: OFL_HEAT_KERNEL (0 CTA-register, 2 warp-independent, 3 two-level) x cells/thread
for cfg in "OFL_HEAT_KERNEL=3" "OFL_HEAT_KERNEL=2 OFL_HEAT_R=16"; do
  echo "== $cfg"; env $cfg python scripts/bench_configs.py --only heat 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin)['config2_heat']; print({k:(v['ms_total'],v['parity_2^20_T1000_bitexact']) for k,v in d.items() if k.startswith('tb')}, d['schedules_agree_bitexact'])"
done
OFL_HEAT_KERNEL=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k heat 2>&1 | tail -2
python scripts/bench_configs.py --only transfer 2>/dev/null
