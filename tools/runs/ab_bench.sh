# usage: bash tools/runs/ab_bench.sh VAR  -> bench with VAR=1 (default) and VAR=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
for v in 1 0 1; do
  env $1=$v timeout 600 python bench.py --no-cpu > gpurun_out/bench_$1_$v.json 2> gpurun_out/bench_$1_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$1_$v.json'));print('$1=$v', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['approx_residual_E'])"
done
