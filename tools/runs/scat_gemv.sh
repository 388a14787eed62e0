python -m pytest tests/test_scattering.py tests/test_gpu_solver.py -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
ncu --set full --clock-control none --import-source on -k regex:k_dgemv_n -c 1 -o gpurun_out/ncu_gemv python tools/gemv_bench.py > gpurun_out/ncu_gemv.log 2>&1
