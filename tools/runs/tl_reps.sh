REPS=6 python tools/timeline.py 1024 > gpurun_out/timeline_pool.txt 2>&1
