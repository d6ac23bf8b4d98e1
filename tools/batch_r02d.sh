# Round-2 batch d: the cleaned library -- GPU suite, bench line, ncu evidence of the final C3 and C4 kernels.
mkdir -p gpurun_out
timeout 5400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 --durations=20 > gpurun_out/gpu_tests_r02d.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_r02d.log
python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02d.json 2> gpurun_out/bench_ref_r02d.err
python tools/run_c3.py --iters 3 > gpurun_out/plain_c3d.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c3full_r02d python tools/run_c3.py --iters 3 > gpurun_out/ncu_c3_r02d.log 2>&1
echo "ncu c3 rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_ncu_plain_d.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02d.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_r02d.log 2>&1
echo "ncu launches rc=$?"
python tools/run_c4.py --iters 3 > gpurun_out/plain_c4d.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c4full_r02d python tools/run_c4.py --iters 3 > gpurun_out/ncu_c4_r02d.log 2>&1
echo "ncu c4 rc=$?"
python tools/bench_c4.py --steps 3 > gpurun_out/c4_balanced_r02d.json 2> gpurun_out/c4d.err
python tools/sweep_c5.py > gpurun_out/c5_sweep_r02d.json 2> gpurun_out/c5d.err
python tools/bench_modes.py > gpurun_out/modes_r02d.json 2> gpurun_out/modesd.err
echo done
