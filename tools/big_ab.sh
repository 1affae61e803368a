L=paper_1911_06895_b200/lib
for r in 1 2; do
python tools/team_probe.py | sed "s/^/base /"
for v in b512 b384 b256; do DS_LIB=$L/libdsssp_$v.so python tools/team_probe.py | sed "s/^/$v /"; done
done
