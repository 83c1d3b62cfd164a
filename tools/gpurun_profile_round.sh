# Round profile: bench line, ncu full captures of the two hot kernels, launch list.
set -x
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench_rc=$?
timeout 300 python tools/profile_lse.py 2 > gpurun_out/p2.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_tile_kernel<.int.2, .int.8, .int.0' -s 4 -c 1 -o gpurun_out/ncu_lse_sum_r01 python tools/profile_lse.py 2 > gpurun_out/ncu_lse_sum_r01.log 2>&1; echo ncu1=$?
timeout 300 python tools/profile_lse.py 3 > gpurun_out/p3.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_mma_kernel' -s 1 -c 1 -o gpurun_out/ncu_block_mma_r01 python tools/profile_lse.py 3 > gpurun_out/ncu_block_r01.log 2>&1; echo ncu2=$?
timeout 600 python bench.py --steps 3 --warmup 1 --no-ttt > gpurun_out/bench_small_r01.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 1 --no-ttt > gpurun_out/ncu_launch_r01.log 2>&1; echo ncu3=$?
