timeout 900 python -m pytest tests/test_gpu_compressed.py -x -q > gpurun_out/gpu_compressed_k.log 2>&1; echo rc=$? >> gpurun_out/gpu_compressed_k.log
timeout 900 python tools/compressed_run.py 256 512 1024 > gpurun_out/compressed_run_k.log 2>&1; echo rc=$? >> gpurun_out/compressed_run_k.log
