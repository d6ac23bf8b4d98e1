# Round-2 GPU batch (one B200): bench line, probes, fixtures, sweeps, then the GPU suite.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
./tools/_dsmem_probe > gpurun_out/dsmem_probe.json 2>&1
python tools/dump_replay_fixture.py gpurun_out/gpu_replay_c3.npz > gpurun_out/replay.log 2>&1
python tools/sweep_c5.py > gpurun_out/c5_sweep_r02.json 2> gpurun_out/c5.err
python tools/bench_c4.py --steps 3 > gpurun_out/c4_balanced_r02.json 2> gpurun_out/c4.err
python tools/bench_c4.py --steps 3 --plan rows > gpurun_out/c4_rows_r02.json 2>> gpurun_out/c4.err
python tools/bench_c4.py --steps 3 --rng reference > gpurun_out/c4_ref_r02.json 2>> gpurun_out/c4.err
python tools/bench_modes.py > gpurun_out/modes_r02.json 2> gpurun_out/modes.err
timeout 5400 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=25 > gpurun_out/gpu_tests_r02.log 2>&1
tail -5 gpurun_out/gpu_tests_r02.log
