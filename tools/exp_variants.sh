for v in base cpi2; do
  RMAT_LIB=paper_1905_03525_b200/_build/exp_$v.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "multi_stream or variants" 2>&1 | tail -1
  RMAT_LIB=paper_1905_03525_b200/_build/exp_$v.so python bench.py --no-cpu --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value']/1e9, d['oracle_check'])"
done
