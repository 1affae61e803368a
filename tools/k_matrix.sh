for d in 0.1 0.25 0.05; do
 for k in 1 2 4 8; do
  if [ "$d" = "0.05" ] && [ "$k" -gt 2 ]; then continue; fi
  if [ "$d" = "0.1" ] && [ "$k" -gt 4 ]; then continue; fi
  DS_LEX=1 DS_LEX_K=$k python bench.py --delta $d --steps 3 --warmup 2 --no-cpu-baseline --no-dropin --no-e2e --no-sweep --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('delta', $d, 'k', $k, round(d['value'],1))"
 done
done
