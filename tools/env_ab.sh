# same-run A/B of env settings on the current build (R-MAT 24 probe, R-MAT 18)
L=paper_1911_06895_b200/lib
run() { local n=$1; shift; env DS_LIB=$L/libdsssp_base.so "$@" python tools/team_probe.py | sed "s/^/$n r24 /"; env DS_LIB=$L/libdsssp_base.so "$@" python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$n /"; }
for r in 1 2; do for spec in "$@"; do run $spec; done; done
