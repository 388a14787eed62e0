timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for old in 0 1; do
VF_QRCP_OLD=$old VF_ID_SPLIT=1 VF_PROF=1 timeout 600 python tools/stage_profile.py --n 1024 --reps 1 > gpurun_out/prof_qrcp$old.txt 2>&1
done
grep small_qrcp gpurun_out/prof_qrcp*.txt
