set -x
python tools/tune_lse.py 4 5 12 13 2>&1 | tail -5
python tools/tune_lse.py 200 201 202 203 2>&1 | tail -4
timeout 300 python tools/profile_lse.py 2 > gpurun_out/p2b.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:pts_tile_kernel<.int.2, .int.8, .int.0' -s 4 -c 1 -o gpurun_out/ncu_lse_sum_r01b python tools/profile_lse.py 2 > gpurun_out/ncu_lse_sum_r01b.log 2>&1; echo ncu1=$?
