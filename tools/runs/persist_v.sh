timeout 900 python -m pytest tests/test_persist.py tests/test_gpu_compressed.py tests/test_gpu_solver.py -q > gpurun_out/gpu_persist_v.log 2>&1; echo rc=$? >> gpurun_out/gpu_persist_v.log
