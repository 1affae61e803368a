# bench throughput vs concurrency (device-resident value only), one line per run
Q="--no-e2e --no-cpu-baseline --no-sweep --no-dropin --no-python-ref --no-clocks"
for c in "$@"; do python bench.py $Q --concurrency $c --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, round(d['value'],1), round(d['solver']['kernel_ms_min'],2), round(d['solver']['kernel_ms_max'],2), d['parity'] if 'parity' in d else '')"; done
