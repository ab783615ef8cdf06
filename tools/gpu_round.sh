# Full round check: build, smoke, gpu tests, quick timings, bench, reference arm, launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 300 python tools/quick_time.py 2>&1 | tail -20
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 120 -c 120 --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
python tools/launches.py gpurun_out/launches_100m.csv
