python -m paper_2507_01021_b200.build > /dev/null
python scripts/encode_profile.py whisper-large-v3 12 > gpurun_out/encprof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_encode_launches_lv3.csv python scripts/encode_profile.py whisper-large-v3 12 > gpurun_out/encprof_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm|attn_tcgen05" -s 230 -c 8 -o gpurun_out/r02_encoder_lv3 python scripts/encode_profile.py whisper-large-v3 12 > gpurun_out/encprof_ncu2.log 2>&1
tail -2 gpurun_out/encprof_ncu2.log
