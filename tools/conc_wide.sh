# batch throughput vs concurrency and wide-window knobs at the current defaults (R-MAT 24, delta 0.1)
for t in 2 3 4 5 6 8; do python tools/pool_probe.py 24 0.1 4 $t | sed "s/^/T=$t /"; done
for a in "DS_WIDE_ALL=0 DS_WIDE_G0=8" "DS_WIDE_ALL=0 DS_WIDE_G0=32" "DS_WIDE_FRAC=0.5" "DS_WIDE_FRAC=0.1" "DS_LEX_PER=1.0" "DS_LEX_PER=2.0"; do
  env $a python tools/pool_probe.py 24 0.1 8 4 | sed "s/^/$a /"
done
