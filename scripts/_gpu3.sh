python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_whisper.py tests/test_gpu_large_v3.py -q -x -p no:cacheprovider 2>&1 | tail -4
python __graft_entry__.py smoke 2>&1 | tail -2
for f in 8 16 24 32; do
  echo "first=$f"; timeout 300 python bench.py --steps 3 --warmup 3 --no-stages --latency-users 0 --no-cpu-baseline --first-encode-batch $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1))"
done
for e in 16 32; do
  echo "encode_batch=$e first=16"; timeout 300 python bench.py --steps 3 --warmup 3 --no-stages --latency-users 0 --no-cpu-baseline --first-encode-batch 16 --encode-batch $e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1))"
done
