python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
timeout 300 python tools/quick_time.py 2>&1 | tail -20
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 90 -c 90 --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
