# ncu full capture of the subtree kernel (100M float3 RR)
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:${KNAME:-subtree_rr} -s ${SKIP:-0} -c 1 -o gpurun_out/${OUT:-subrr} python tools/one_build.py ${N:-100000000} 3 ${MODE:-rr} ${KIND:-uniform} 1 > gpurun_out/prof7.log 2>&1
tail -2 gpurun_out/prof7.log
