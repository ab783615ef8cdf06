python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for K in sel_hist sel_filter sel_select; do
ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o gpurun_out/$K python tools/one_build.py 100000000 3 rr uniform 1 > /dev/null 2>&1
done
ls gpurun_out
