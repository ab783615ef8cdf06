# Config 5 evidence: widest clustered 100M bench line (per-kernel classes), launch list, subtree_sel source lines
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 5 --warmup 3 --mode widest --dist clustered --no-cpu-baseline > gpurun_out/bench_widest.log 2>&1; tail -1 gpurun_out/bench_widest.log > gpurun_out/bench_widest.json
tail -1 gpurun_out/bench_widest.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['e2e']['value']); [print(k, v['ms_per_build'], v.get('achieved_gbs')) for k, v in d['kernels'].items()]"
L=$(python tools/one_build.py 100000000 3 widest clustered 1 | awk '/launches per build/{print $4}')
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_widest.csv python tools/one_build.py 100000000 3 widest clustered 2 > gpurun_out/profw1.log 2>&1
python tools/launches.py gpurun_out/launches_widest.csv > gpurun_out/launches_widest.txt
ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/subsel python tools/one_build.py 100000000 3 widest clustered 1 > gpurun_out/profw2.log 2>&1
python tools/ncu_lines.py gpurun_out/subsel.ncu-rep 40 > gpurun_out/subsel_lines.txt 2>&1
cat gpurun_out/launches_widest.txt
