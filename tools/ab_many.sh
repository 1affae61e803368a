# same-run A/B over several library builds (R-MAT 24, R-MAT 18, grid 2048)
L=paper_1911_06895_b200/lib
run() { # name, lib, env...
  local n=$1 lib=$2; shift 2
  env DS_LIB=$L/libdsssp_$lib.so "$@" python tools/team_probe.py | sed "s/^/$n r24 /"
  env DS_LIB=$L/libdsssp_$lib.so "$@" python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$n /"
}
for r in 1 2; do
for v in $@; do run $v $v; done
done
for v in $@; do DS_LIB=$L/libdsssp_$v.so python tools/trace_grid.py 2048 | head -1 | sed "s/^/$v /"; done
