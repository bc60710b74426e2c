python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err; tail -2 gpurun_out/bench_v8.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_v8.json").read())
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "launches", d["gpu_launches"])
print("roof", d["roofline"]["frac"], d["roofline"]["avg_launch_ms"], d["roofline"]["kv_stream_only_frac"])
for k,v in d["stages"].items():
    if isinstance(v, dict): print(k, round(v["frac"],3), round(v["ms"],3), v.get("fp32_frac"))
print("lat", d["latency"]["multiplexed"]["p50_ms"], d["latency"]["multiplexed"]["p95_ms"], d["latency"]["sequential_single_user"]["p95_ms"])
print("cpu", d["cpu_baseline"]["value"], "clocks", d["clocks"])
P
timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/r02_step_trace_lv3_v8.json 2>&1
