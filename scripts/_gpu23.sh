python -m paper_2507_01021_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_ctc.py tests/test_gpu_whisper.py -q -s -x -p no:cacheprovider -k "ctc or refill" 2>&1 | grep -E "seg |passed|failed|Error|assert" | head -20
time (timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err); tail -c 1500 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
