python -m paper_2507_01021_b200.build > /dev/null
rm -f gpurun_out/parity_report.jsonl
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -1
