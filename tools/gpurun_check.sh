# Fresh-box check: GPU tests, smoke, default bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_chk.json 2> gpurun_out/bench_chk.err; echo bench_rc=$?
cat gpurun_out/bench_chk.json; tail -5 gpurun_out/bench_chk.err
