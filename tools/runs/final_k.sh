timeout 900 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; echo rc=$? >> gpurun_out/bench_k.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_k.json 2> gpurun_out/bench_ref_k.err
