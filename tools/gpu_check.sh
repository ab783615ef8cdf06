# build, smoke, GPU parity tests, quick timings, per-kernel-class breakdown of the bench
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/quick_time.py 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_check.log 2>&1
tail -1 gpurun_out/bench_check.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['e2e']['value']); [print(k, v['ms_per_build'], v.get('achieved_gbs')) for k, v in d['kernels'].items()]"
