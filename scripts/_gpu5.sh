python -m paper_2507_01021_b200.build > /dev/null
timeout 300 python scripts/step_trace.py whisper-large-v3 64 1 > gpurun_out/trace_tc.json 2>&1
python - <<'P'
import json
d=json.load(open("gpurun_out/trace_tc.json"))
for rows,v in d.items():
    print(rows, v["step_us"], v["by_kind"]["xattn"])
    for r in v["layer0"]:
        if r["k"].endswith("xattn"): print(r)
P
