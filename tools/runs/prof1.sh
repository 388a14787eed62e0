VF_PROF=1 python tools/stage_profile.py --n 1024 > gpurun_out/prof_c.txt 2>&1
