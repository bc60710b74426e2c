python -m paper_2507_01021_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_length_aware.py tests/test_gpu_whisper.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not large_v3" 2>&1 | tail -15
