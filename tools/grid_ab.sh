L=paper_1911_06895_b200/lib
for v in $@; do DS_LIB=$L/libdsssp_$v.so python tools/trace_grid.py 4096 2>/dev/null | head -1 | sed "s/^/$v /"; done
