# reduction grids: CTAs (512 threads) per SM for sum_u32 2^28 and dot_f32 2^31
for c in 1 2 3 4; do
  echo "== OFL_REDUCE_CPS=$c"; OFL_REDUCE_CPS=$c python scripts/bench_configs.py --only sum,dot 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('sum', d['sum_u32']['kernel_ms'], d['sum_u32']['gbs'], d['sum_u32']['bitexact'], '| dot', d['config4_dot']['kernel_ms'], d['config4_dot']['gbs'], d['config4_dot']['rel_err'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sum or dot" 2>&1 | tail -2
