python -m paper_2507_01021_b200.build > /dev/null
for la in 0 1; do echo "LA $la"; LA=$la timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 8 1 2>&1 | head -3; done
