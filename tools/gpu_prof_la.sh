mkdir -p gpurun_out
python tools/prof_cluster.py > gpurun_out/prof_la_plain.log 2>&1; cat gpurun_out/prof_la_plain.log
ncu --set full --import-source on --clock-control none -k regex:dense_cluster_la_kernel -c 1 -o gpurun_out/prof_la_b1 -f \
    python tools/prof_cluster.py > gpurun_out/prof_la_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_la_b1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_la_b1_sass.csv 2>&1
