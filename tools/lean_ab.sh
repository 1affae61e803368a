L=paper_1911_06895_b200/lib
for r in 1 2; do
python tools/team_probe.py | sed "s/^/base /"
DS_BIG_L=4000000 python tools/team_probe.py | sed "s/^/base+L4M /"
for v in lean640 lean512 lean384; do
DS_LIB=$L/libdsssp_$v.so python tools/team_probe.py | sed "s/^/$v /"
DS_LIB=$L/libdsssp_$v.so DS_BIG_L=4000000 python tools/team_probe.py | sed "s/^/$v+L4M /"
DS_LIB=$L/libdsssp_$v.so DS_BIG_L=1000000 DS_BIG_H=1000000 python tools/team_probe.py | sed "s/^/$v+LH1M /"
done; done
