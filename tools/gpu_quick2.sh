python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/quick_time.py 2>&1 | tail -20
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 90 -c 90 --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
./tools/micro/gather
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --csv -k regex:"k_(plain|cg|nc|cv|l2|rel)" ./tools/micro/gather > gpurun_out/micro_gather.csv 2>&1
