# Full GPU suite, smoke, default bench line (with the fp32 leg).
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r2.err
