for v in 2 1; do
VF_QR_UNR=$v VF_ID_SPLIT=1 VF_PROF=1 timeout 600 python tools/stage_profile.py --n 1024 --reps 1 > gpurun_out/prof_qru$v.txt 2>&1
grep "panel_qr" gpurun_out/prof_qru$v.txt | awk '{s+=$2; printf "%s:%s ", substr($1,2,2), $2} END {print " total", s}'
done
VF_QR_UNR=2 timeout 900 python -m pytest tests/test_gpu_id.py tests/test_gpu_solver.py -x -q 2>&1 | tail -1
