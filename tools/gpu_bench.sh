python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -3
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -2
