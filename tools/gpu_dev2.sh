# dev loop: build, smoke, gpu parity tests (select path), quick timings
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -5
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -25
timeout 300 python tools/quick_time.py 2>&1 | tail -20
