# A/B kernel variants: each prebuilt library in $VARIANTS, interleaved, 3 rounds.
VARIANTS=${VARIANTS:-"base"}
for v in $VARIANTS; do
  RMAT_LIB=paper_1905_03525_b200/_build/exp_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "multi_stream or variants" 2>&1 | tail -1
done
for round in 1 2 3; do
  for v in $VARIANTS; do
    RMAT_LIB=paper_1905_03525_b200/_build/exp_$v.so timeout 300 python bench.py --no-cpu --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9, 2), d['oracle_check']['bit_exact'])"
  done
done
