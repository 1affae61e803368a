L=paper_1911_06895_b200/lib
for r in 1 2; do
DS_HEAVY_PULL=0 DS_LIB=$L/libdsssp_hp.so python tools/team_probe.py | sed "s/^/push r24 /"
DS_LIB=$L/libdsssp_hp.so python tools/team_probe.py | sed "s/^/pull r24 /"
DS_HEAVY_PULL=0 DS_LIB=$L/libdsssp_hp.so python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/push /"
DS_LIB=$L/libdsssp_hp.so python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/pull /"
done
DS_LIB=$L/libdsssp_hp.so python tools/trace.py 24 2>&1 | head -8
