# Source-level ncu capture of the widest in-CTA selection kernel
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/subsel10 python tools/one_build.py 100000000 3 widest clustered 1 > gpurun_out/prof10.log 2>&1
python tools/ncu_lines.py gpurun_out/subsel10.ncu-rep 50 > gpurun_out/subsel10_lines.txt 2>&1
head -50 gpurun_out/subsel10_lines.txt
