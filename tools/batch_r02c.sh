# Round-2 batch c (final library): GPU suite, bench line, ncu evidence, sweeps with clocks.
mkdir -p gpurun_out
timeout 5400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 --durations=30 > gpurun_out/gpu_tests_r02c.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_r02c.log
python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
echo "bench rc=$?"
python tools/run_c3.py --iters 3 > gpurun_out/plain_c3c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c3full_r02c python tools/run_c3.py --iters 3 > gpurun_out/ncu_c3_r02c.log 2>&1
echo "ncu c3 rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_ncu_plain_c.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_r02c.log 2>&1
echo "ncu launches rc=$?"
./tools/_dsmem_probe > gpurun_out/dsmem_probe_c.json 2>&1
python tools/sweep_c5.py > gpurun_out/c5_sweep_r02c.json 2> gpurun_out/c5c.err
python tools/bench_c4.py --steps 3 > gpurun_out/c4_balanced_r02c.json 2> gpurun_out/c4c.err
python tools/bench_c4.py --steps 3 --rng reference > gpurun_out/c4_ref_r02c.json 2>> gpurun_out/c4c.err
python tools/bench_modes.py > gpurun_out/modes_r02c.json 2> gpurun_out/modesc.err
echo done
