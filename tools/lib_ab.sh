# same-run A/B of library builds: tools/lib_ab.sh SCALE DELTA NAME...  (lib/libdsssp_NAME.so;
# NAME "main" = lib/libdsssp.so); each build measured twice, interleaved
L=paper_1911_06895_b200/lib
S=$1; D=$2; shift 2
for r in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then f=$L/libdsssp.so; else f=$L/libdsssp_$v.so; fi
  DS_LIB=$f python tools/pool_probe.py $S $D 16 4 | sed "s/^/$v /"
done
done
