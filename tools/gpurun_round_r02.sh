# Round-2 check on the box: GPU tests, smoke, default bench line, the GPU side of the
# full-size parity runs, ncu of the tensor-core block pass and the launch list of a short bench.
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
for cfg in C4 C3; do
  tag=$(echo "$cfg" | tr 'A-Z' 'a-z'); mkdir -p gpurun_out/${tag}_r02
  SKNR_PARITY_CFG=$cfg timeout 600 python tools/full_parity.py gpu > gpurun_out/${tag}_r02/gpu.log 2>&1; echo "gpu $cfg rc=$?"
done
timeout 300 python tools/profile_i8.py > gpurun_out/i8_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_i8w_kernel' -s 1 -c 1 -o gpurun_out/ncu_i8w_r02 python tools/profile_i8.py > gpurun_out/ncu_i8w_r02.log 2>&1
echo "ncu_i8 rc=$?"; cat gpurun_out/i8_plain.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/bench_small_r02.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/ncu_launch_r02.log 2>&1
echo "launch list rc=$?"
