L=paper_1911_06895_b200/lib
run() { local n=$1; shift; env DS_LIB=$L/libdsssp_co.so "$@" python tools/team_probe.py | sed "s/^/$n r24 /"; env DS_LIB=$L/libdsssp_co.so "$@" python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$n /"; }
for r in 1 2; do run default DS_CARVEOUT=-1; run min; run c100 DS_CARVEOUT=100; run c58 DS_CARVEOUT=58; done
