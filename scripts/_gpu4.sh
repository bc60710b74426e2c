python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_whisper.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not large_v3" 2>&1 | tail -4
timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 16 8 1 2>&1 | head -5
timeout 300 python scripts/xattn_compare.py whisper-base 64 16 1 2>&1 | head -3
