# same-run A/B of env settings on the current build (R-MAT 24 probe, R-MAT 18, grid 2048)
L=paper_1911_06895_b200/lib
run() { local n=$1; shift; env DS_LIB=$L/libdsssp_base.so "$@" python tools/team_probe.py | sed "s/^/$n r24 /"; env DS_LIB=$L/libdsssp_base.so "$@" python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$n /"; }
for r in 1 2; do
run default
run small DS_SMALL=1
run smallE4k DS_SMALL=1 DS_LOCAL_E=4096 DS_LOCAL_N=1024
run smallE64k DS_SMALL=1 DS_LOCAL_E=65536 DS_LOCAL_N=8192
done
