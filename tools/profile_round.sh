# round-end profile set (run under gpurun): bench without ncu, launch list of the same command,
# one --set full capture of an R-MAT 24 solve and one of the grid solve, exported to CSV
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks --no-dropin --no-sweep"
$B > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/prof_launches.csv $B > gpurun_out/prof_ncu_bench.log 2>&1
python tools/one_source.py > gpurun_out/prof_one.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -c 1 -f -o gpurun_out/r2c_prof python tools/one_source.py > gpurun_out/prof_ncu_one.log 2>&1
ncu -i gpurun_out/r2c_prof.ncu-rep --page raw --csv > gpurun_out/r2c_raw.csv
python tools/one_grid.py > gpurun_out/prof_grid.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:sssp_persistent -c 1 -f -o gpurun_out/r2c_grid python tools/one_grid.py > gpurun_out/prof_ncu_grid.log 2>&1
ncu -i gpurun_out/r2c_grid.ncu-rep --page raw --csv > gpurun_out/r2c_grid_raw.csv
cat gpurun_out/prof_one.log gpurun_out/prof_grid.log; tail -c 400 gpurun_out/prof_bench.json
