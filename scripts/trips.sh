python -c "from paper_2009_10863_b200.build import build; build()" > /dev/null
for t in 0 1 2 4 8 16; do echo "MIN_TRIPS=$t"; IG_MIN_TRIPS=$t timeout 300 python scripts/bench_sweep.py --sizes 100000,1000000,2097152,10000000 --ms 8 --steps 20 2>&1 | grep "^| [0-9]"; done
