set -x
Q="--no-e2e --no-cpu-baseline --no-sweep --no-dropin --no-python-ref"
python tools/trace.py 24 > gpurun_out/d1_trace24.txt 2>&1
for c in 4 4 2 8; do python bench.py $Q --concurrency $c --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, d['value'], d['solver']['kernel_ms_min'], d['solver']['kernel_ms_max'])" >> gpurun_out/d1_conc.txt; done
DS_TRACE=0 timeout 300 python tools/trace_grid.py 4096 > gpurun_out/d1_tracegrid.txt 2>&1
timeout 300 python tools/cta_balance.py 24 > gpurun_out/d1_cta.txt 2>&1
