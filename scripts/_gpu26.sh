python -m paper_2507_01021_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_whisper.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not large_v3" 2>&1 | tail -2
timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 16 8 1 2>&1 | head -5
timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/trace_x4.json 2>&1
python - <<'P'
import json
d=json.load(open("gpurun_out/trace_x4.json"))
for rows,v in d.items():
    print(rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items() if k in ("xattn","xo","self","fc1")})
P
