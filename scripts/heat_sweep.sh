# register-blocked heat kernel: cells per thread x temporal block
for r in 8 16 32; do
  echo "== OFL_HEAT_R=$r"; OFL_HEAT_R=$r python scripts/bench_configs.py --only heat 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin)['config2_heat']; print({k:(v['ms_total'],v['parity_2^20_T1000_bitexact']) for k,v in d.items() if k.startswith('tb')}, d['schedules_agree_bitexact'])"
done
