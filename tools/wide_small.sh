# wide windows beyond the headline: small R-MAT graphs (lex ksub 1 forced on) and the grid
for s in 18 20 22; do
  DS_WIDE=0 python tools/batch_probe.py $s | grep -E "conc=(1|8):" | sed "s/^/off /"
  DS_LEX1_MIN_NNZ=0 python tools/batch_probe.py $s | grep -E "conc=(1|8):" | sed "s/^/wide /"
done
python tools/trace_grid.py 2048 | head -8 | sed "s/^/small-kernel /"
DS_SMALL=0 DS_LEX1_MIN_NNZ=0 DS_WIDE_FORCE=1 DS_WIDE_G0=62 DS_WIDE_HI=1e18 python tools/trace_grid.py 2048 | head -8 | sed "s/^/wide62 /"
DS_SMALL=0 DS_LEX1_MIN_NNZ=0 DS_WIDE_FORCE=1 DS_WIDE_G0=16 DS_WIDE_HI=1e18 DS_WIDE_LO=0 python tools/trace_grid.py 2048 | head -8 | sed "s/^/wide16 /"
