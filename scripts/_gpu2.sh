python -m paper_2507_01021_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_whisper.py -q -x -k "streaming or batch_invariance or overlapped" -p no:cacheprovider 2>&1 | tail -5
timeout 300 python scripts/xattn_compare.py whisper-large-v3 > gpurun_out/xattn_cmp_lv3.log 2>&1; cat gpurun_out/xattn_cmp_lv3.log | head -12
timeout 300 python scripts/xattn_compare.py whisper-base 64 32 16 8 > gpurun_out/xattn_cmp_base.log 2>&1; cat gpurun_out/xattn_cmp_base.log | head -6
XA_MODE=0 timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/r02_step_trace_lv3.json 2> gpurun_out/step_trace.err; tail -2 gpurun_out/step_trace.err
python - <<'P'
import json
d=json.load(open("gpurun_out/r02_step_trace_lv3.json"))
for rows,v in d.items(): print(rows, v["step_us"], {k:(x["n"],x["gap_us"],x["span_us"]) for k,x in v["by_kind"].items()})
P
