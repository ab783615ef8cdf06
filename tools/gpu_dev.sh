set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30
timeout 300 python tools/quick_time.py 2>&1 | tail -20
