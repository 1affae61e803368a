# same-run A/B of two library builds: bash tools/ab2.sh <libA> <libB>
L=paper_1911_06895_b200/lib
for r in 1 2; do
for v in $1 $2; do
DS_LIB=$L/libdsssp_$v.so python tools/team_probe.py | sed "s/^/$v r24 /"
DS_LIB=$L/libdsssp_$v.so python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$v /"
done; done
for v in $1 $2; do DS_LIB=$L/libdsssp_$v.so python tools/trace_grid.py 2048 | head -1 | sed "s/^/$v /"; done
