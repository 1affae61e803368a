# wide-window thresholds on R-MAT 24 (same build, same run): entry size, settled share, first window
D=${1:-0.1}
run() { env "$@" python tools/pool_probe.py 24 $D 8 4 | sed "s/^/$* /"; }
run DS_WIDE=0
run DS_WIDE_ENTER=8e6 DS_WIDE_FRAC=0.125 DS_WIDE_G0=2
run DS_WIDE_ENTER=3e7 DS_WIDE_FRAC=0.25 DS_WIDE_G0=2
run DS_WIDE_ENTER=3e7 DS_WIDE_FRAC=0.25 DS_WIDE_G0=8
run DS_WIDE_ENTER=1e9 DS_WIDE_FRAC=0.25 DS_WIDE_G0=4
run DS_WIDE_ENTER=1e9 DS_WIDE_FRAC=0.25 DS_WIDE_G0=16
run DS_WIDE_ENTER=1e9 DS_WIDE_FRAC=0.25 DS_WIDE_G0=64 DS_WIDE_HI=1e9
run DS_WIDE_ENTER=1e9 DS_WIDE_FRAC=1.0 DS_WIDE_G0=4
run DS_WIDE_ENTER=1e9 DS_WIDE_FRAC=0.25 DS_WIDE_G0=8 DS_WIDE_LO=1e7 DS_WIDE_HI=1e8
