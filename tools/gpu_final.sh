# Round evidence (final): ncu captures first (their traffic / issue summaries feed the
# bench lines), then tests, bench lines (RR headline, widest config 5, reference arm), 1B config 4
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
# RR 100M uniform: launch list + DRAM traffic per kernel class, full captures
L=$(python tools/one_build.py 100000000 3 rr uniform 1 | awk '/launches per build/{print $4}')
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
python tools/launches.py gpurun_out/launches_100m.csv > gpurun_out/launches_100m.txt
python tools/ncu_traffic.py gpurun_out/launches_100m.csv profiles/ncu_traffic.json > /dev/null
ncu --set full --clock-control none --import-source on -k regex:sel_part -s 4 -c 1 -o gpurun_out/part python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/subrr python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sel_filter -s 6 -c 1 -o gpurun_out/filter python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof4.log 2>&1
python tools/ncu_issue.py gpurun_out/subrr.ncu-rep profiles/ncu_issue_subtree.json > /dev/null
# widest 100M clustered
L=$(python tools/one_build.py 100000000 3 widest clustered 1 | awk '/launches per build/{print $4}')
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_widest.csv python tools/one_build.py 100000000 3 widest clustered 2 > gpurun_out/profw1.log 2>&1
python tools/launches.py gpurun_out/launches_widest.csv > gpurun_out/launches_widest.txt
python tools/ncu_traffic.py gpurun_out/launches_widest.csv profiles/ncu_traffic_widest.json > /dev/null
ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/subsel python tools/one_build.py 100000000 3 widest clustered 1 > gpurun_out/profw2.log 2>&1
python tools/ncu_issue.py gpurun_out/subsel.ncu-rep profiles/ncu_issue_subtree_widest.json > /dev/null
cp profiles/ncu_traffic.json profiles/ncu_traffic_widest.json profiles/ncu_issue_subtree.json profiles/ncu_issue_subtree_widest.json gpurun_out/
# tests, benches
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json; cut -c1-300 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json; cut -c1-300 gpurun_out/bench_ref.json
timeout 900 python bench.py --steps 5 --warmup 3 --mode widest --dist clustered > gpurun_out/bench_widest.log 2>&1; tail -1 gpurun_out/bench_widest.log > gpurun_out/bench_widest.json; cut -c1-300 gpurun_out/bench_widest.json
timeout 300 python tools/quick_time.py > gpurun_out/quick_time.txt 2>&1; cat gpurun_out/quick_time.txt
timeout 600 python tools/robust_time.py > gpurun_out/robust_time.txt 2>&1; cat gpurun_out/robust_time.txt
timeout 900 python tools/big_build.py 1000000000 clustered 3 > gpurun_out/big_1b.log 2>&1; tail -1 gpurun_out/big_1b.log | cut -c1-400
cat gpurun_out/launches_100m.txt gpurun_out/launches_widest.txt
