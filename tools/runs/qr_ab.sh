for v in 1 0; do
VF_QR_NT128=$v VF_ID_SPLIT=1 VF_PROF=1 timeout 600 python tools/stage_profile.py --n 1024 --reps 1 > gpurun_out/prof_qr$v.txt 2>&1
grep "panel_qr" gpurun_out/prof_qr$v.txt | awk '{printf "%s %s | ", substr($1,2,2), $2}'; echo
done
VF_QR_NT128=1 timeout 900 python -m pytest tests/test_gpu_id.py tests/test_gpu_solver.py -x -q 2>&1 | tail -2
