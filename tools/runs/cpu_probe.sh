(cat /sys/fs/cgroup/cpu.max; nproc; python -c "import os; print(len(os.sched_getaffinity(0)))"; cat /proc/cpuinfo | grep -c processor; cat /sys/fs/cgroup/cpu.stat) > gpurun_out/cpu_probe.txt 2>&1
OPENBLAS_NUM_THREADS=1 OMP_NUM_THREADS=1 MKL_NUM_THREADS=1 REPS=6 python tools/timeline.py 1024 > gpurun_out/timeline_1thr.txt 2>&1
cat /sys/fs/cgroup/cpu.stat >> gpurun_out/cpu_probe.txt 2>&1
