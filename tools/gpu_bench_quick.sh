mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_f4.json 2> gpurun_out/bench_f4.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_f4.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_f4.json").read().strip().splitlines()[-1])
print("value", d["value"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"])
for r in d.get("selection_and_async", []): print(r)
for r in d.get("other_configs", []): print({k: r.get(k) for k in ("workload","sweeps","time_to_eps_ms","frac","status")})
for e in d.get("paper_envs", []): print(e["env"], [(x["b"], x["sweeps"], round(x["time_to_eps_ms"],2)) for x in e["vi"]])
print(d.get("clocks"))
PY
