mkdir -p gpurun_out
python tools/prof_sparse_c4.py > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sparse_solver_kernel -c 1 -o gpurun_out/prof_c4 -f python tools/prof_sparse_c4.py > gpurun_out/c4_ncu.log 2>&1
echo "c4 rc=$?"
python tools/prof_sparse_c3.py > gpurun_out/c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sparse_solver_kernel -c 1 -o gpurun_out/prof_c3 -f python tools/prof_sparse_c3.py > gpurun_out/c3_ncu.log 2>&1
echo "c3 rc=$?"
cat gpurun_out/c4_plain.log gpurun_out/c3_plain.log
