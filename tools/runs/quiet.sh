REPS=6 python tools/timeline.py 1024 > gpurun_out/timeline_quiet.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_quiet.json 2> gpurun_out/bench_quiet.err
