L=paper_1911_06895_b200/lib
DS_TIMEOUT_S=20 DS_LIB=$L/libdsssp_x1.so python tools/trace.py 24 2>&1 | head -20
