python -m paper_2507_01021_b200.build > /dev/null
echo "192"; timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 8 1 2>&1 | head -4
echo "128"; DM_LIB=_variants/lib128/libdictamux_b200.so timeout 300 python scripts/xattn_compare.py whisper-large-v3 64 32 8 1 2>&1 | head -4
