mkdir -p gpurun_out
for N in 1024 1448 2048; do python tools/c4size.py $N; done > gpurun_out/c4size.txt 2>&1
for N in 1024 1448 2048; do ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:sparse_solver_kernel -s 1 -c 1 python tools/c4size.py $N 2>&1 | grep -E "dram__|lts__|gpu__time|N="; done >> gpurun_out/c4size.txt
cat gpurun_out/c4size.txt
