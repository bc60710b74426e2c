python -m paper_2507_01021_b200.build > /dev/null
timeout 300 python scripts/run_timeline.py 24 64 2>&1 | tail -30
timeout 300 python scripts/run_timeline.py 16 16 2>&1 | tail -30 | head -9
timeout 300 python scripts/run_timeline.py 8 8 2>&1 | tail -30 | head -9
timeout 600 python bench.py --steps 3 --warmup 3 --latency-users 0 --no-cpu-baseline > gpurun_out/bench_v6.json 2> gpurun_out/bench_v6.err; tail -2 gpurun_out/bench_v6.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_v6.json').read()); print(d['value'], d['roofline'])"
