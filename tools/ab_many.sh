# same-run A/B over several library builds / env settings (R-MAT 24 and 18)
L=paper_1911_06895_b200/lib
run() { # name, lib, env...
  local n=$1 lib=$2; shift 2
  env DS_LIB=$L/libdsssp_$lib.so "$@" python tools/team_probe.py | sed "s/^/$n r24 /"
  env DS_LIB=$L/libdsssp_$lib.so "$@" python tools/batch_probe.py 18 | grep "conc=1:" | sed "s/^/$n /"
}
for r in 1 2; do
run base base
run nohandoff base DS_BIG_H=100000000000
run bigH16M base DS_BIG_H=16000000
run c512 c512
run pipe pipe
run t1024 t1024
run t640 t640
done
