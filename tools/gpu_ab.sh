# A/B of an in-CTA kernel switch: parity tests, then timings with the switch off and on.
# usage: bash tools/gpu_ab.sh ENVVAR
V=${1:-LBKD_BUCKET}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6
echo "== $V=0"; env $V=0 timeout 300 python tools/quick_time.py 2>&1 | tail -6
echo "== default"; timeout 300 python tools/quick_time.py 2>&1 | tail -6
timeout 300 python tools/robust_time.py 2>&1 | tail -12
