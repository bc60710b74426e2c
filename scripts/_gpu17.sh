python -m paper_2507_01021_b200.build > /dev/null
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 8 1 2>&1 | head -4
timeout 900 python bench.py > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err; tail -2 gpurun_out/bench_v5.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_v5.json").read())
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "launches", d["gpu_launches"])
print("roof", d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])
for k,v in d["stages"].items():
    if isinstance(v, dict): print(k, round(v["frac"],3), round(v["ms"],3), v.get("fp32_frac"))
print("lat", d["latency"]["multiplexed"]["p50_ms"], d["latency"]["multiplexed"]["p95_ms"], d["latency"]["sequential_single_user"]["p95_ms"])
print("cpu", d["cpu_baseline"]["value"], "clocks", d["clocks"])
P
