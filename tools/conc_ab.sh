L=paper_1911_06895_b200/lib
for v in $@; do DS_LIB=$L/libdsssp_$v.so python tools/batch_probe.py 24 | sed "s/^/$v /"; done
