python -m paper_2507_01021_b200.build > /dev/null
for la in 0 1; do
LA=$la timeout 300 python scripts/step_trace.py whisper-large-v3 64 8 > gpurun_out/trace_la$la.json 2>&1
python - $la <<'P'
import json,sys
d=json.load(open(f"gpurun_out/trace_la{sys.argv[1]}.json"))
for rows,v in d.items():
    print("LA", sys.argv[1], rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items() if k in ("xattn","xo","self")})
P
done
