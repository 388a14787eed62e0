timeout 900 python -m pytest tests/test_scattering.py tests/test_gpu_compressed.py -x -q > gpurun_out/gpu_scat_t.log 2>&1; echo rc=$? >> gpurun_out/gpu_scat_t.log
