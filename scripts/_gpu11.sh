python -m paper_2507_01021_b200.build > /dev/null
python scripts/decode_kernel_probe.py 64 0,7,1 whisper-large-v3 > gpurun_out/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cross_attn|gemv_kernel|self_attn" -s 3 -c 12 -o gpurun_out/r02_decode_lv3 python scripts/decode_kernel_probe.py 64 0,7,1 whisper-large-v3 > gpurun_out/probe_ncu.log 2>&1
tail -3 gpurun_out/probe_ncu.log; cat gpurun_out/probe_plain.log
