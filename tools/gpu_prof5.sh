python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 40 -c 1 -o gpurun_out/pass0 python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hist_kernel -s 5 -c 1 -o gpurun_out/hist python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof5.log 2>&1
