set -x
python -m paper_2507_01021_b200.build > /dev/null
timeout 300 python scripts/step_trace.py whisper-large-v3 64 32 8 1 > gpurun_out/r02_step_trace_lv3.json 2> gpurun_out/step_trace.err
tail -3 gpurun_out/step_trace.err
timeout 300 python scripts/decode_kernel_probe.py 64 0 whisper-large-v3 --nostep > gpurun_out/xprobe_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cross_attn -s 2 -c 1 -o gpurun_out/r02_xattn_lv3 python scripts/decode_kernel_probe.py 64 0 whisper-large-v3 --nostep > gpurun_out/xprobe_ncu.log 2>&1
tail -3 gpurun_out/xprobe_ncu.log
timeout 300 python bench.py --profile > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/r02_launches_lv3.csv python bench.py --profile > gpurun_out/prof_ncu.log 2>&1
tail -3 gpurun_out/prof_ncu.log
ls -la gpurun_out
