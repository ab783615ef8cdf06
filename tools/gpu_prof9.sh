# Source-level ncu capture of the in-CTA subtree kernel + clustered RR timing
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/subrr9 python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/prof9.log 2>&1
python tools/ncu_lines.py gpurun_out/subrr9.ncu-rep 60 > gpurun_out/subrr9_lines.txt 2>&1
python tools/ncu_issue.py gpurun_out/subrr9.ncu-rep gpurun_out/ncu_issue9.json > /dev/null 2>&1
head -70 gpurun_out/subrr9_lines.txt
cat gpurun_out/ncu_issue9.json
