python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python bench.py --latency-users 0 --no-cpu-baseline > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; tail -2 gpurun_out/bench_v9.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_v9.json").read())
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
print("LA", d["length_aware_opt_in"])
print("roof", d["roofline"]["frac"])
for k,v in d["stages"].items():
    if isinstance(v, dict): print(k, round(v["frac"],3), round(v["ms"],3))
P
