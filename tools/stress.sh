timeout 600 python tools/stress.py 30 65536 8192 2>&1 | tail -3
F2_LIB=tools/lib_split.so timeout 600 python tools/stress.py 30 65536 8192 2>&1 | tail -3
timeout 600 python tools/stress.py 15 65536 65536 2>&1 | tail -3
