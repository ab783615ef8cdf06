python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
