set -x
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 4000 gpurun_out/bench.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 3 --warmup 3 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/bench_torchrun1.json 2>&1; echo torchrun rc=$?; tail -c 600 gpurun_out/bench_torchrun1.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?; tail -c 800 gpurun_out/bench_ref.json
