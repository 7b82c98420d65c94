for rep in 1 2 3 4; do timeout 600 python tools/race.py 20 2>&1 | tail -1; done
F2_SPLIT_EARLY=1 timeout 600 python tools/race.py 20 2>&1 | tail -1
timeout 600 python tools/t3.py 65536 10 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
