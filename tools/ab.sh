# A/B kernel variants on one GPU (run under gpurun).  Each prebuilt library
# paper_1905_03525_b200/_build/exp_<v>.so (tools/build_variants.py) is first
# checked bit-exact (GPU parity + fuzz suites), then timed interleaved:
# C3 bench.py (k_packed<16,smem>) x ROUNDS, and C4 parts (tools/bench_c4.py) if C4=1.
# usage: VARIANTS="base v1 v2" [C3V="..."] [C4V="..."] [ROUNDS=3] [TESTS=1] [ENV_v1="X=1"] bash tools/ab.sh
# (ENV_<variant>: extra environment for that variant's runs, e.g. the oracle's
# RMAT_FAST_CTR when the variant changes the fast path's counter layout)
VARIANTS=${VARIANTS:-"base"}
C3V=${C3V:-$VARIANTS}
C4V=${C4V:-}
ROUNDS=${ROUNDS:-3}
LIBD=paper_1905_03525_b200/_build
if [ "${TESTS:-1}" = 1 ]; then
  for v in $VARIANTS; do
    eval "venv=\${ENV_$v:-}"
    r=$(env $venv RMAT_LIB=$LIBD/exp_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1)
    echo "tests $v: $r"
  done
fi
for round in $(seq $ROUNDS); do
  for v in $C3V; do
    eval "venv=\${ENV_$v:-}"
    env $venv RMAT_LIB=$LIBD/exp_$v.so timeout 300 python bench.py --no-cpu --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $v', round(d['value']/1e9, 2), d['oracle_check']['bit_exact'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
if [ -n "$C4V" ]; then
  for round in 1 2; do
    for v in $C4V; do
      eval "venv=\${ENV_$v:-}"
      env $venv RMAT_LIB=$LIBD/exp_$v.so timeout 300 python tools/bench_c4.py --steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $v', round(d['value']/1e9, 2))"
    done
  done
fi
if [ -n "${REFV:-}" ]; then
  for v in $REFV; do
    eval "venv=\${ENV_$v:-}"
    env $venv RMAT_LIB=$LIBD/exp_$v.so timeout 300 python tools/ref_c3_time.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ref $v', {k: round(x/1e9, 2) for k, x in d.items()})"
  done
fi
