# ksub x delta with wide windows on (pool probe: single-solve ms and 4-in-flight batch GTEPS)
for d in 0.1 0.25 0.05; do
 for k in 1 2 4 8; do
  DS_LEX=1 DS_LEX_K=$k python tools/pool_probe.py 24 $d 8 4 | sed "s/^/delta $d k $k /"
 done
done
