# long call: C4 oracle trajectories (both accept modes) on the host cores in the background;
# GPU-side evidence in the foreground (timings here are not bench numbers)
SECS=${SECS:-3300} JOBS="C4:stable:8 C4:literal:8" CHUNK=2 bash tools/gpurun_oracle_bg.sh \
  'timeout 1200 python tools/accept_modes.py 12 > gpurun_out/accept_modes6.log 2>&1' \
  'timeout 600 python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/bench_small6.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/ncu_launch6.log 2>&1; echo launches=$?' \
  'bash tools/gpurun_ncu.sh 4 pts_mma2_kernel 1 ncu_block_rs_v2_r02'
