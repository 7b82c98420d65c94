F2_LIB=tools/lib_split.so timeout 900 python tools/race.py 40 2>&1 | tail -1
F2_LIB=tools/lib_split.so timeout 900 python tools/race.py 40 2>&1 | tail -1
timeout 900 python tools/race.py 30 2>&1 | tail -1
F2_LIB=tools/lib_split.so timeout 300 python tools/t3.py 65536 10 2>&1 | tail -1
timeout 300 python tools/t3.py 65536 10 2>&1 | tail -1
