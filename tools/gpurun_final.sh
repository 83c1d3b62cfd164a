# Round-end refresh: GPU tests, smoke, bench line, launch list of the no-ttt bench command.
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/bench_small_final.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/ncu_launch_final.log 2>&1
echo launch_rc=$?
