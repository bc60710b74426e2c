python -m paper_2507_01021_b200.build > /dev/null
timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 16 8 1 2>&1 | head -5
