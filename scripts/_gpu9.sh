python -m paper_2507_01021_b200.build > /dev/null
for m in 0 1 2; do
DM_GV_ROWPLAN=$m timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 1 > gpurun_out/trace_gv$m.json 2>&1
echo "mode $m"
python - $m <<'P'
import json,sys
d=json.load(open(f"gpurun_out/trace_gv{sys.argv[1]}.json"))
for rows,v in d.items():
    print(rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items() if k in ("qkv","o","xq","fc1","fc2","lm_head","xattn")})
P
done
