set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_j.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_j.log 2>&1; echo rc=$? >> gpurun_out/smoke_j.log
timeout 900 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo rc=$? >> gpurun_out/bench_j.err
