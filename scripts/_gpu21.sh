python -m paper_2507_01021_b200.build > /dev/null
for i in 1 2 3; do
timeout 600 python bench.py --steps 5 --warmup 3 --latency-users 0 --no-cpu-baseline --no-stages 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1), d['gpu_launches'])"
done
timeout 300 python scripts/run_timeline.py 24 64 2>&1 | grep -v Warn | head -12
