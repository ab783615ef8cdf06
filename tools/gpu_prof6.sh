# ncu: launch list of one 100M float3 build + full captures of the partition and subtree kernels
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
N=$(python tools/one_build.py 1000 3 rr uniform 1 2>/dev/null | awk '/launches per build/{print $4}')
python tools/one_build.py 100000000 3 rr uniform 1 | tail -1
L=$(python tools/one_build.py 100000000 3 rr uniform 1 | awk '/launches per build/{print $4}')
echo "launches per build: $L"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
python tools/launches.py gpurun_out/launches_100m.csv
ncu --set full --clock-control none --import-source on -k regex:sel_part -s 3 -c 1 -o gpurun_out/part python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:subtree_rr -c 1 -o gpurun_out/subrr python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof3.log 2>&1
ls -la gpurun_out
