# wide windows A/B on R-MAT 24: off vs on at several thresholds (same build, same run)
#   tools/wide_ab.sh [DELTA]
D=${1:-0.1}
for r in 1 2; do
  DS_WIDE=0 python tools/pool_probe.py 24 $D 8 4 | sed "s/^/wide=0 /"
  python tools/pool_probe.py 24 $D 8 4 | sed "s/^/wide=default /"
done
