timeout 900 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo rc=$? >> gpurun_out/bench_i.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_256.csv python bench.py --n 256 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
