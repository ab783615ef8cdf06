ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 90 -c 90 --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:subtree -s 1 -c 1 -o gpurun_out/subtree python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:onesweep -s 60 -c 2 -o gpurun_out/pass python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rekey -s 18 -c 1 -o gpurun_out/rekey python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof4.log 2>&1
ls -la gpurun_out
