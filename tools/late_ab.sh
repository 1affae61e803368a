L=paper_1911_06895_b200/lib
for r in 1 2; do
for v in base late; do
if [ $v = base ]; then E=""; else E="DS_LIB=$L/libdsssp_$v.so"; fi
env $E python tools/team_probe.py | sed "s/^/$v r24 /"
env $E python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$v /"
done; done
DS_LIB=$L/libdsssp_late.so timeout 600 python -m pytest tests -m gpu -x -q -k "block_local or handoff or rmat18 or batch or corpus or rmat20" 2>&1 | tail -1
