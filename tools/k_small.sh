for s in 18 20 22; do
  python tools/batch_probe.py $s | grep -E "conc=(1|8):" | sed "s/^/k1 /"
  DS_LEXK_MIN_NNZ=0 python tools/batch_probe.py $s | grep -E "conc=(1|8):" | sed "s/^/kauto /"
done
