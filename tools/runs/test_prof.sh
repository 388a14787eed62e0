python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
VF_PROF=1 python tools/stage_profile.py --n 1024 > gpurun_out/prof_d.txt 2>&1
