timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_l.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_l.log
timeout 900 python tools/compressed_run.py 256 512 1024 > gpurun_out/compressed_run_l.log 2>&1; echo rc=$? >> gpurun_out/compressed_run_l.log
