# r02 evidence: the bench line, the launch list of the bench's GPU arm, and one
# ncu --set full capture of the headline kernel (b = 1000, 20 sweeps)
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/prof_dense.py 1000 20 > gpurun_out/prof_dense_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_tma_kernel -c 1 -o gpurun_out/prof_dense_r02 -f \
    python tools/prof_dense.py 1000 20 > gpurun_out/prof_dense_ncu.log 2>&1
echo "ncu full rc=$?"
