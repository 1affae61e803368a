# SM-sharing A/B: batch throughput of block-shape variants (lib/libdsssp_NAME.so; "main" = the
# default build) at several concurrencies.  Narrow CTAs let the T concurrent grids of a batch
# co-reside on every SM instead of taking SM-disjoint slices.
#   tools/share_ab.sh SCALE DELTA "NAME:T1,T2" ...
L=paper_1911_06895_b200/lib
S=$1; D=$2; shift 2
for r in 1 2; do
for spec in "$@"; do
  v=${spec%%:*}; ts=${spec#*:}
  if [ "$v" = main ]; then f=$L/libdsssp.so; else f=$L/libdsssp_$v.so; fi
  for t in ${ts//,/ }; do
    DS_LIB=$f python tools/pool_probe.py $S $D 8 $t | sed "s/^/$v T=$t /"
  done
done
done
