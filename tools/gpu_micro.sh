nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather tools/micro/gather.cu
/tmp/gather
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --csv -k regex:"k_(plain|cg|nc|cv|l2|rel)" /tmp/gather > gpurun_out/micro_gather.csv 2>&1
