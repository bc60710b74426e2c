python -m paper_2507_01021_b200.build > /dev/null
for cfg in "8 8" "16 16" "8 16" "4 8" "12 12" "8 8" "16 32"; do
set -- $cfg
echo "first $1 eb $2"; timeout 600 python bench.py --steps 5 --warmup 3 --latency-users 0 --no-cpu-baseline --no-stages --first-encode-batch $1 --encode-batch $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1))"
done
