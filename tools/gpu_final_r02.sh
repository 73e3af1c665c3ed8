# end-of-round evidence: bench line (+ reference arm), launch list of the GPU arm
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_final2.json 2> gpurun_out/bench_ref_final2.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/plain_launch2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/ncu_launch2.log 2>&1
echo "launch list rc=$?"
