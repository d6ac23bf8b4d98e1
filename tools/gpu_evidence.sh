# GPU evidence batch (one B200, under gpurun): the GPU suite, the bench line, ncu captures of the C3 and C4 kernels (each after its plain run exits 0), C4 / C5 / modes with clocks.
mkdir -p gpurun_out
timeout 5400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 --durations=20 > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/run_c3.py --iters 3 > gpurun_out/plain_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c3full python tools/run_c3.py --iters 3 > gpurun_out/ncu_c3.log 2>&1
echo "ncu c3 rc=$?"
# the reports are large (gpurun_out/ is capped at 64 MiB): export what tools/ncu_summary.py and tools/sass_mix.py read, drop the report
ncu -i gpurun_out/c3full.ncu-rep --page raw --csv > gpurun_out/c3_raw.csv 2>/dev/null
ncu -i gpurun_out/c3full.ncu-rep --page source --print-source sass --csv > gpurun_out/c3_sass.csv 2>/dev/null
rm -f gpurun_out/c3full.ncu-rep
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_ncu_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
python tools/run_c4.py --iters 3 > gpurun_out/plain_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_packed -s 2 -c 1 -f -o gpurun_out/c4full python tools/run_c4.py --iters 3 > gpurun_out/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
ncu -i gpurun_out/c4full.ncu-rep --page raw --csv > gpurun_out/c4_raw.csv 2>/dev/null
ncu -i gpurun_out/c4full.ncu-rep --page source --print-source sass --csv > gpurun_out/c4_sass.csv 2>/dev/null
rm -f gpurun_out/c4full.ncu-rep
python tools/bench_c4.py --steps 3 > gpurun_out/c4_balanced.json 2> gpurun_out/c4.err
python tools/sweep_c5.py > gpurun_out/c5_sweep.json 2> gpurun_out/c5.err
python tools/bench_modes.py > gpurun_out/modes.json 2> gpurun_out/modes.err
echo done
