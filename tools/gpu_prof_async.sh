mkdir -p gpurun_out
python tools/prof_async.py 20 > gpurun_out/prof_async_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/prof_async_plain.log
ncu --set full --clock-control none --import-source on -k regex:dense_async_tma_kernel -c 1 -o gpurun_out/prof_async_r02 -f \
    python tools/prof_async.py 20 > gpurun_out/prof_async_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_async_ncu.log
