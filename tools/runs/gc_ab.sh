VF_GC_PAUSE=0 REPS=4 python tools/timeline.py 1024 > gpurun_out/timeline_gc_on.txt 2>&1
REPS=4 python tools/timeline.py 1024 > gpurun_out/timeline_gc_off.txt 2>&1
python bench.py --no-cpu > gpurun_out/bench_gc.json 2> gpurun_out/bench_gc.err
