mkdir -p gpurun_out
python tools/prof_sparse_c4.py eval > gpurun_out/c4e_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sparse_solver_kernel -c 1 -o gpurun_out/prof_c4e -f python tools/prof_sparse_c4.py eval > gpurun_out/c4e_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/c4e_plain.log
