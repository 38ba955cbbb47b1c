timeout 300 python tools/debug_parity.py 9 150003 blobs 3 1000000 2>&1 | tail -40
