timeout 900 python -m pytest tests/test_gpu_compressed.py -x -q > gpurun_out/gpu_ti_s.log 2>&1; echo rc=$? >> gpurun_out/gpu_ti_s.log
