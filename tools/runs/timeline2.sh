VF_ID_SPLIT=0 python tools/timeline.py 1024 > gpurun_out/timeline_nosplit.txt 2>&1
python tools/timeline.py 1024 > gpurun_out/timeline_split.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python bench.py --no-cpu > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err
