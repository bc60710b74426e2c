python -m paper_2507_01021_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_whisper.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not large_v3" 2>&1 | tail -2
timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/trace_pl.json 2>&1
python - <<'P'
import json
d=json.load(open("gpurun_out/trace_pl.json"))
for rows,v in d.items():
    print(rows, v["step_us"], {k:round(x["span_us"]) for k,x in v["by_kind"].items()}, "gaps", round(sum(x["gap_us"] for x in v["by_kind"].values())))
P
timeout 600 python bench.py --steps 3 --warmup 3 --latency-users 0 --no-cpu-baseline --no-stages > gpurun_out/bench_v7.json 2> gpurun_out/bench_v7.err; tail -2 gpurun_out/bench_v7.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_v7.json').read()); print(d['value'], d['e2e']['value'])"
