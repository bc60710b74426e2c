python -m paper_2507_01021_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_whisper.py tests/test_gpu_large_v3.py -q -x -p no:cacheprovider 2>&1 | tail -2
for sp in 4 10; do
echo "fc1 splits $sp"
DM_FC1_SPLITS=$sp timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/trace_f$sp.json 2>&1
python - $sp <<'P'
import json,sys
d=json.load(open(f"gpurun_out/trace_f{sys.argv[1]}.json"))
for rows,v in d.items():
    print(rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items() if k in ("fc1","gelu","fc2","ln1","ln3")})
P
done
