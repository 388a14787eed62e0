timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for v in 1 0; do
VF_SELECT_HH=$v VF_ID_SPLIT=1 VF_PROF=1 timeout 600 python tools/stage_profile.py --n 1024 --reps 1 > gpurun_out/prof_sel$v.txt 2>&1
grep "^n=\|profiled" gpurun_out/prof_sel$v.txt
done
python - <<'PY'
import re,collections
for v in (1,0):
    agg=collections.defaultdict(float)
    for line in open(f'gpurun_out/prof_sel{v}.txt'):
        m=re.match(r'(L(\d\d)\.)?(\S+)\s+([\d.]+) ms\s+\((\d+)\)',line)
        if m: agg[m.group(3)]+=float(m.group(4))
    print(v, {k: round(agg[k],1) for k in ['id.setup+select','id.panel_qr','id.gemm_W','id.small_qrcp']})
PY
