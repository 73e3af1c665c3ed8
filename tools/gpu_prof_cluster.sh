mkdir -p gpurun_out
python tools/prof_cluster.py > gpurun_out/cl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_cluster_kernel -c 1 -o gpurun_out/prof_cluster -f python tools/prof_cluster.py > gpurun_out/cl_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/cl_plain.log
