# Round-2 GPU batch b: the GPU suite, then the ncu evidence (each only after its plain run exits 0).
mkdir -p gpurun_out
timeout 5400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 --durations=30 > gpurun_out/gpu_tests_r02.log 2>&1
echo "tests rc=$?"
python tools/run_c3.py --iters 3 > gpurun_out/plain_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c3full_r02 python tools/run_c3.py --iters 3 > gpurun_out/ncu_c3_r02.log 2>&1
echo "ncu c3 rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_ncu_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_r02.log 2>&1
echo "ncu launches rc=$?"
python tools/run_c4.py --iters 3 > gpurun_out/plain_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c4full_r02 python tools/run_c4.py --iters 3 > gpurun_out/ncu_c4_r02.log 2>&1
echo "ncu c4 rc=$?"
tail -3 gpurun_out/gpu_tests_r02.log
