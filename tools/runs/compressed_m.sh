timeout 900 python -m pytest tests/test_gpu_compressed.py -x -q > gpurun_out/gpu_compressed_m.log 2>&1; echo rc=$? >> gpurun_out/gpu_compressed_m.log
timeout 900 python tools/compressed_bench.py > gpurun_out/compressed_bench_m.json 2> gpurun_out/compressed_bench_m.err; echo rc=$? >> gpurun_out/compressed_bench_m.err
