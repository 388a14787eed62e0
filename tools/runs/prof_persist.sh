python -m pytest tests/test_persist.py -x -q > gpurun_out/persist_tests.log 2>&1; echo rc=$? >> gpurun_out/persist_tests.log
timeout 600 python tools/persist_bench.py --n 512 > gpurun_out/persist_512.json 2> gpurun_out/persist.err
VF_PROF=1 timeout 600 python tools/stage_profile.py --n 1024 --reps 2 > gpurun_out/prof_1024.txt 2>&1
