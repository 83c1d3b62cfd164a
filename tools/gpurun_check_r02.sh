# Round-2 check on a fresh box: GPU tests, smoke, default bench line.
set -x
nproc > gpurun_out/host_nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
