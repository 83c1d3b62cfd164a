set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_r01_a.json 2> gpurun_out/bench_r01_a.err; echo bench_rc=$?
cat gpurun_out/bench_r01_a.json; tail -5 gpurun_out/bench_r01_a.err
timeout 300 python tools/profile_lse.py 2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_tile_kernel<2, 4, 0, 0>' -s 5 -c 1 -o gpurun_out/lse_sum_r01 python tools/profile_lse.py 2 > gpurun_out/ncu_lse.log 2>&1; echo ncu_rc=$?
timeout 300 python tools/profile_lse.py 3 > gpurun_out/prof_plain3.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_tile_kernel<2, 1, 2, 32>' -s 1 -c 1 -o gpurun_out/block_r01 python tools/profile_lse.py 3 > gpurun_out/ncu_block.log 2>&1; echo ncu3_rc=$?
timeout 600 python bench.py --steps 3 --warmup 1 --no-ttt > gpurun_out/bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 1 --no-ttt > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
tail -3 gpurun_out/ncu_lse.log gpurun_out/ncu_block.log gpurun_out/ncu_launch.log
