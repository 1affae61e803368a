L=paper_1911_06895_b200/lib
for r in 1 2; do
DS_LIB=$L/libdsssp_base.so python tools/team_probe.py | sed "s/^/base r24 /"
DS_LIB=$L/libdsssp_base.so DS_BIG_H=100000000000 python tools/team_probe.py | sed "s/^/nohandoff r24 /"
DS_LIB=$L/libdsssp_base.so DS_BIG_H=16000000 python tools/team_probe.py | sed "s/^/bigH16M r24 /"
DS_LIB=$L/libdsssp_pipe.so python tools/team_probe.py | sed "s/^/pipe r24 /"
done
