python -m paper_2507_01021_b200.build > /dev/null
for la in 0 1; do LA=$la timeout 300 python scripts/run_timeline.py 12 12 2>&1 | grep -v -i warn | head -20; done
