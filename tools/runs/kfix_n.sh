timeout 900 python -m pytest tests/test_gpu_id.py tests/test_gpu_compressed.py -x -q > gpurun_out/gpu_kfix_n.log 2>&1; echo rc=$? >> gpurun_out/gpu_kfix_n.log
