# end-of-round measurement set (run under gpurun); large ncu reports stay in /tmp on the box
set -x
T=${1:-r02c}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_ncu_list.log 2>&1; echo list rc=$?
ncu --set full --clock-control none --import-source on -k regex:'leaf_|tri_canon' -o /tmp/${T}_c1_full python tools/prof_c1.py > gpurun_out/${T}_ncu_full.log 2>&1; echo full rc=$?
ncu -i /tmp/${T}_c1_full.ncu-rep --page raw --csv > gpurun_out/${T}_c1_full_raw.csv 2>/dev/null; echo raw rc=$?
python bench.py --config 0 --no-cpu-baseline > gpurun_out/${T}_bench_config0.json 2>gpurun_out/${T}_c0.err; echo c0 rc=$?
python bench.py --config 2 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/${T}_bench_config2.json 2>gpurun_out/${T}_c2.err; echo c2 rc=$?
