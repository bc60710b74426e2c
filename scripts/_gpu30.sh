python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_vad.py -q -x -p no:cacheprovider 2>&1 | tail -3
