for v in "" "OFL_REDUCE_PERSISTENT=1"; do
  echo "== $v"; env $v python scripts/bench_configs.py --only sum,dot 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['sum_u32']['kernel_ms'], d['sum_u32']['gbs'], d['sum_u32']['bitexact'], d['config4_dot']['kernel_ms'], d['config4_dot']['gbs'], d['config4_dot']['rel_err'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "sum or dot" 2>&1 | tail -2
