set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; tail -3 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1; tail -c 400 gpurun_out/bench_ref_final.log
python bench.py --matrix > gpurun_out/c5_matrix_final.jsonl 2> gpurun_out/c5_matrix_final.err; tail -3 gpurun_out/c5_matrix_final.jsonl | cut -c1-300
mkdir -p gpurun_out/r2cap
timeout 400 ncu --set full --import-source on --clock-control none -k regex:sweep_scan_kernel -s 3 -c 1 -o gpurun_out/r2cap/c5s2 python bench.py --steps 1 --warmup 3 --no-solvers --no-e2e --no-cpu > gpurun_out/r2cap/c5s2.log 2>&1
ncu -i gpurun_out/r2cap/c5s2.ncu-rep --page raw --csv > gpurun_out/r2cap/c5s2_raw.csv
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2cap/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-solvers --no-e2e --no-cpu > gpurun_out/r2cap/bench_launches.log 2>&1
ls gpurun_out/r2cap
