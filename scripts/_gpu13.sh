python -m paper_2507_01021_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_whisper.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not large_v3" 2>&1 | tail -2
for c in 0 1; do
DM_XA_CLUSTER=$c timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/trace_lean$c.json 2>&1
echo "cluster=$c"
python - $c <<'P'
import json,sys
d=json.load(open(f"gpurun_out/trace_lean{sys.argv[1]}.json"))
for rows,v in d.items():
    print(rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items()})
P
done
timeout 600 python bench.py --steps 5 --warmup 3 --latency-users 0 --no-cpu-baseline > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; tail -2 gpurun_out/bench_v4.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_v4.json").read())
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
print("roof", d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])
for k,v in d["stages"].items():
    if isinstance(v, dict): print(k, round(v["frac"],3), round(v["ms"],3), v.get("fp32_frac"))
P
