python -m paper_2507_01021_b200.build > /dev/null
timeout 600 python scripts/enc_kernels.py whisper-large-v3 12 24 64 2>&1 | grep -v Warn
